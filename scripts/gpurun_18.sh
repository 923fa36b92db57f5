#!/bin/bash
# panel trace + full ncu capture of a mid-run trailing GEMM and panel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GBLA_PANEL_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace18.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain18.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:k_modgemm_tc|k_panel' -s 120 -c 4 -o gpurun_out/prof18 $CMD > gpurun_out/ncu_full18.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full18.log

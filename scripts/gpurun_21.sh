#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain21.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:k_panel2|k_modgemm_tc|k_sweep' -s 60 -c 4 -o gpurun_out/prof21 $CMD > gpurun_out/ncu_full21.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full21.log

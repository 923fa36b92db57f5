#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain9.log 2>&1 && \
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_sweep_step|k_modgemm_tc|k_panel" -s 120 -c 6 -o gpurun_out/prof9 $CMD > gpurun_out/ncu9.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu9.log

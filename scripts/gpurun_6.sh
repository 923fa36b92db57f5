#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain6.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_panel|k_sweep|k_modgemm_tc|k_update_tc" -c 7 -o gpurun_out/prof6 $CMD > gpurun_out/ncu6.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu6.log

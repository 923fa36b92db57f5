#!/bin/bash
# source-level ncu of one dense c3 panel (blocked LU) and one c1 panel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:k_panel2 -s 20 -c 1 -o gpurun_out/panel_c3b python bench.py --config c3 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_p3.log 2>&1
timeout 900 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:k_panel2 -s 30 -c 1 -o gpurun_out/panel_c1b python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_p1.log 2>&1

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:k_panel2 -s 30 -c 1 -o gpurun_out/panel57 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu57.log 2>&1

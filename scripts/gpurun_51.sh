#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python bench.py --steps 6 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/b_on.log 2>&1
GBLA_KERNEL_TIMERS= timeout 600 python bench.py --steps 6 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b_off.log 2>&1

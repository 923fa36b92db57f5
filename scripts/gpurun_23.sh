#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GBLA_ECH_TIMELINE=40 timeout 600 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/tl.log 2>&1
GBLA_KERNEL_TIMERS= timeout 600 python bench.py --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b_notimers.log 2>&1
GBLA_NO_LOOKAHEAD=1 timeout 600 python bench.py --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b_nola.log 2>&1

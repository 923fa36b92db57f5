#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GBLA_KERNEL_TIMERS= GBLA_ECH_TIMELINE=400 timeout 900 python bench.py --config c2 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/tl2.log 2>&1

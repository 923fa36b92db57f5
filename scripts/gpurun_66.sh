#!/bin/bash
# echelon chain timeline on c1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GBLA_ECH_TIMELINE=10 timeout 600 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/tl_c1.log 2>&1

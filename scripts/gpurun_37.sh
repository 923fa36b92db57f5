#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for w in 8 16; do
  GBLA_EPI_WARPS=$w timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_$w.log 2>&1
  GBLA_EPI_WARPS=$w timeout 600 python bench.py --config c3 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3_$w.log 2>&1
done
GBLA_NO_LOOKAHEAD=1 timeout 600 python bench.py --config c3 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3_nola.log 2>&1

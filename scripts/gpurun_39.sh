#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for i in 1 2 3; do
timeout 600 python bench.py --steps 8 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_$i.log 2>&1
done

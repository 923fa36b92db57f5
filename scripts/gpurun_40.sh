#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2 3; do
timeout 600 python bench.py --steps 8 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_$i.log 2>&1
done
timeout 900 python bench.py --config c2 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b2.log 2>&1

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x --durations=0 > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
timeout 600 python bench.py --config c3 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --config c2 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1

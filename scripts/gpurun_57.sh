#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
GBLA_SP=4 timeout 900 python -m pytest tests -m gpu -q -x -k "not fullsize" > gpurun_out/pytest_sp4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sp4.log
GBLA_SP=4 timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_sp4.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1.log 2>&1
GBLA_SP=4 timeout 600 python bench.py --config c3 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3_sp4.log 2>&1
timeout 600 python bench.py --config c3 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3.log 2>&1
GBLA_SP=4 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k c3 > gpurun_out/pytest_fs_sp4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fs_sp4.log

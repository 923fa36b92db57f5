#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --config c2 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b2_sp4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_fs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fs.log
timeout 1200 python bench.py --config c4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b4_sp4.log 2>&1

#!/bin/bash
# B tiles of the next window only on the look-ahead chain: parity, bench, timeline
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1.log 2>&1
GBLA_ECH_TIMELINE=6 timeout 600 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/tl_c1.log 2>&1
timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3" > gpurun_out/pytest_fs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fs.log

#!/bin/bash
# sweep two-step look-ahead (GBLA_SWEEP_PAIRS=1): parity on every shape, bench c1/c3/c2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GBLA_SWEEP_PAIRS=1 timeout 300 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_pairs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pairs.log
GBLA_SWEEP_PAIRS=1 timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_pairs.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1.log 2>&1
GBLA_SWEEP_PAIRS=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3_pairs.log 2>&1
GBLA_SWEEP_PAIRS=1 timeout 400 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3 or c2" > gpurun_out/pytest_fs_pairs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fs_pairs.log

#!/bin/bash
# memory query for X-tile batches (c4 timed step after a warmup), tight K11 timers, fill_rows fmod32
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1.log 2>&1
timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b4.log 2>&1

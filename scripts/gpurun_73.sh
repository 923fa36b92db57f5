#!/bin/bash
# padded shared row strides (conflict-free fragments): parity, trace c1/c3, bench c1/c3
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
GBLA_PANEL_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_c1.log 2>&1
GBLA_PANEL_TRACE=1 timeout 600 python bench.py --config c3 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_c3.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1.log 2>&1
timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3.log 2>&1

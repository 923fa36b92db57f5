#!/bin/bash
# panel: two-barrier rounds: parity, trace, bench c1 (+ lumode 0 parity on c3 shapes)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
GBLA_PANEL_LU=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "scaled or engines or c0_full or without_lookahead" > gpurun_out/pytest_lu0.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lu0.log
GBLA_PANEL_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_c1.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1.log 2>&1

#!/bin/bash
# blocked dense LU (GBLA_PANEL_LU=3): parity (incl. dense random D), trace c3, bench c3/c1, fullsize c3
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
GBLA_PANEL_TRACE=1 timeout 600 python bench.py --config c3 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_c3.log 2>&1
timeout 600 python bench.py --config c3 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3" > gpurun_out/pytest_fs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fs.log

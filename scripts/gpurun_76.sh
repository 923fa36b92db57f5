#!/bin/bash
# fixed 8-lane phase F (c3 dense panels); main-stream chain schedule (vs GBLA_LA_SIDE); HBM roofline of K11
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
GBLA_LA_MAIN=1 timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -k "c0_full or scaled or ref_mode" > gpurun_out/pytest_side.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_side.log
timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1.log 2>&1
GBLA_LA_SIDE=1 timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_side.log 2>&1
GBLA_ECH_TIMELINE=6 timeout 300 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/tl_c1.log 2>&1
GBLA_PANEL_TRACE=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_c3.log 2>&1
timeout 300 python bench.py --config c3 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3.log 2>&1
timeout 400 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3" > gpurun_out/pytest_fs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fs.log

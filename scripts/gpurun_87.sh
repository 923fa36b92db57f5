#!/bin/bash
# main-stream chain (GBLA_LA_MAIN) with the fused window step and the leads before the rest: parity + c1 both ways
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GBLA_LA_MAIN=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c0_full or scaled or ref_mode or c1_full or edge or random_suite_new or window" > gpurun_out/pytest_lamain.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lamain.log
GBLA_LA_MAIN=1 timeout 240 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_lamain.log 2>&1
timeout 240 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1.log 2>&1
GBLA_LA_MAIN=1 timeout 240 python bench.py --config c3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3_lamain.log 2>&1

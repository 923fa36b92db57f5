#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x --durations=0 > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain25.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:k_sweep|k_modgemm_ws' -s 4 -c 3 -o gpurun_out/prof25 $CMD > gpurun_out/ncu_full25.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full25.log

#!/bin/bash
# memory query that empties torch's cache first (c4 full-size test after the other tests), alloc
# callback returning NULL on OOM; full ncu capture of a K11 trailing (rest) launch
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/f_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_pytest_gpu.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_modgemm_ws -s 43 -c 1 -o gpurun_out/f_trailing python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/f_ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/f_ncu_full.log

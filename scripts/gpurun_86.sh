#!/bin/bash
# window step + lead scan in one launch (grid barrier): parity, bench c1 vs GBLA_WIN_LEAD=0
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 240 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1.log 2>&1
GBLA_WIN_LEAD=0 timeout 240 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_nolead.log 2>&1
GBLA_ECH_TIMELINE=6 timeout 240 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/tl.log 2>&1

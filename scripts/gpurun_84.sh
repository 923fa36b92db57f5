#!/bin/bash
# fused window step (GBLA_WIN_FUSED=1): parity (bounded spin: a failure cannot hang), bench c1 both ways
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GBLA_WIN_FUSED=1 timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "c0_full or scaled or ref_mode or c1_full or edge or random_suite_new" > gpurun_out/pytest_win.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_win.log
GBLA_WIN_FUSED=1 timeout 240 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_win.log 2>&1
timeout 240 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1.log 2>&1
GBLA_WIN_FUSED=1 GBLA_ECH_TIMELINE=6 timeout 240 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/tl_win.log 2>&1

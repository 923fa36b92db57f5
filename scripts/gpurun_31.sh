#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in a b c d; do
  case $v in
    a|b) unset GBLA_NO_LOOKAHEAD;;
    c|d) export GBLA_NO_LOOKAHEAD=1;;
  esac
  timeout 600 python bench.py --steps 6 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
done

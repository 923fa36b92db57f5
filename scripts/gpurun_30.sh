#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in a b c; do
  case $v in
    a) export GBLA_KERNEL_TIMERS=1; unset GBLA_KT_MAIN_ONLY;;
    b) export GBLA_KERNEL_TIMERS=1; export GBLA_KT_MAIN_ONLY=1;;
    c) export GBLA_KERNEL_TIMERS=; unset GBLA_KT_MAIN_ONLY;;
  esac
  timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
done

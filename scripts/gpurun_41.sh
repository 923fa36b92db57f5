#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in pf2 pf1; do
  if [ $v = pf1 ]; then export GBLA_EPI_PF1=1; else unset GBLA_EPI_PF1; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_$v.log 2>&1
  timeout 600 python bench.py --config c3 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3_$v.log 2>&1
  timeout 900 python bench.py --config c2 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b2_$v.log 2>&1
done
unset GBLA_EPI_PF1
GBLA_NO_LOOKAHEAD=1 timeout 900 python bench.py --config c2 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b2_nola.log 2>&1

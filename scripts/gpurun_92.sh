#!/bin/bash
# lead scan grid: 8 vs 4 blocks per SM
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in 8 4 16; do
  GBLA_LEAD_BPS=$v timeout 240 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/lead_$v.log 2>&1
done
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c0_full or scaled or c1_full" > gpurun_out/pytest_lead.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lead.log

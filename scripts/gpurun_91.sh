#!/bin/bash
# knob sweep on c1 with the final build
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for kv in "X=0" "GBLA_PANEL_CAP=96" "GBLA_PANEL_CAP=112" "GBLA_EPI_WARPS=16" "GBLA_PANEL_LU=1"; do
  env $kv timeout 240 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/knob_${kv}.log 2>&1
done

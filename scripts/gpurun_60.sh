#!/bin/bash
# panel phase trace + echelon timeline (c1, c3)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GBLA_PANEL_TRACE=1 GBLA_ECH_TIMELINE=12 timeout 600 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_c1.log 2>&1
GBLA_PANEL_TRACE=1 timeout 600 python bench.py --config c3 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_c3.log 2>&1

#!/bin/bash
# rounds vs pivot steps per chunk (GBLA_PANEL_LU 0/1/2) on c1 and c3; parity of the default
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for m in 0 1 2; do
GBLA_PANEL_LU=$m timeout 600 python bench.py --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b1_lu$m.log 2>&1
GBLA_PANEL_LU=$m timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3_lu$m.log 2>&1
done
GBLA_PANEL_LU=0 GBLA_PANEL_TRACE=1 timeout 600 python bench.py --config c3 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_c3_lu0.log 2>&1
GBLA_PANEL_LU=0 GBLA_PANEL_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_c1_lu0.log 2>&1

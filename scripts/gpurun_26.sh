#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GBLA_NO_LOOKAHEAD=1 GBLA_PANEL_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_nola.log 2>&1
GBLA_PANEL_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/trace_la.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain26.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:k_sweep' -c 1 -o gpurun_out/prof26s $CMD > gpurun_out/ncu26s.log 2>&1 ; \
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:k_modgemm_ws|k_panel2' -s 100 -c 3 -o gpurun_out/prof26g $CMD > gpurun_out/ncu26g.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu26g.log

mkdir -p gpurun_out/pk
GBLA_PANEL_TRACE=1 timeout 300 python bench.py --config c1 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pk/trace_c1.log 2>&1; grep "panel2 trace" gpurun_out/pk/trace_c1.log | tail -1
GBLA_PANEL_TRACE=1 timeout 300 python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pk/trace_c2.log 2>&1; grep "panel2 trace" gpurun_out/pk/trace_c2.log | tail -1
GBLA_ECH_TIMELINE=12 timeout 300 python bench.py --config c1 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pk/tl_c1.log 2>&1; grep "gbla timeline" gpurun_out/pk/tl_c1.log | tail -12
ENV_SWEEP_STEPS=4 timeout 300 python scripts/env_sweep.py c1 "" "GBLA_PANEL_CAP=96" "GBLA_PANEL_CAP=64" "GBLA_PANEL_CAP=112" > gpurun_out/pk/c1.jsonl 2>gpurun_out/pk/c1.err; cut -c1-260 gpurun_out/pk/c1.jsonl
ENV_SWEEP_STEPS=2 timeout 600 python scripts/env_sweep.py c2 "" "GBLA_PANEL_CAP=96" "GBLA_PANEL_CAP=64" > gpurun_out/pk/c2.jsonl 2>gpurun_out/pk/c2.err; cut -c1-260 gpurun_out/pk/c2.jsonl
tail -n 2 gpurun_out/pk/*.err

mkdir -p gpurun_out/c3k
GBLA_PANEL_TRACE=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c3k/trace.log 2>&1; grep "panel2 trace" gpurun_out/c3k/trace.log | tail -1
GBLA_ECH_TIMELINE=24 timeout 300 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c3k/tl.log 2>&1; grep "gbla timeline" gpurun_out/c3k/tl.log | tail -24
ENV_SWEEP_STEPS=2 timeout 900 python scripts/env_sweep.py c3 "" "GBLA_SP=2" "GBLA_SP=1" "GBLA_SP=3" "GBLA_PANEL_CAP=96" "GBLA_PANEL_CAP=64" > gpurun_out/c3k/c3.jsonl 2>gpurun_out/c3k/c3.err; cut -c1-300 gpurun_out/c3k/c3.jsonl; tail -n 2 gpurun_out/c3k/c3.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_sweep -c 1 -o gpurun_out/c3k/ncu_sweep_c2 python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c3k/ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -2 gpurun_out/c3k/ncu_full.log

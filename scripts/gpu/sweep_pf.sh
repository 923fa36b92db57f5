mkdir -p gpurun_out/pf
ENV_SWEEP_STEPS=2 timeout 600 python scripts/env_sweep.py c2 "" "GBLA_SWEEP_EXP=4" "" "GBLA_SWEEP_EXP=4" > gpurun_out/pf/c2.jsonl 2>gpurun_out/pf/c2.err; cut -c1-200 gpurun_out/pf/c2.jsonl

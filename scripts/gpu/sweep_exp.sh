mkdir -p gpurun_out/se
ENV_SWEEP_STEPS=2 timeout 900 python scripts/env_sweep.py c2 "" "GBLA_SWEEP_EXP=2" "GBLA_SWEEP_EXP=3" "GBLA_SWEEP_EXP=1" "GBLA_SWEEP_EXP=2,GBLA_SWEEP_GROUP=16" > gpurun_out/se/c2b.jsonl 2>gpurun_out/se/c2b.err; cut -c1-200 gpurun_out/se/c2b.jsonl; tail -n 3 gpurun_out/se/c2b.err

mkdir -p gpurun_out/tl3
GBLA_REF_FULLSCAN=1 GBLA_ECH_TIMELINE=8 timeout 300 python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/tl3/full.log 2>&1; grep "gbla timeline" gpurun_out/tl3/full.log | tail -6
GBLA_ECH_TIMELINE=8 timeout 300 python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/tl3/pre.log 2>&1; grep "gbla timeline" gpurun_out/tl3/pre.log | tail -6

mkdir -p gpurun_out/tl2
GBLA_ECH_TIMELINE=30 timeout 300 python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/tl2/tl_c2.log 2>&1; grep "gbla timeline" gpurun_out/tl2/tl_c2.log | tail -30

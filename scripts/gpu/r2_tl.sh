mkdir -p gpurun_out/tl
for c in c2 c1; do
GBLA_ECH_TIMELINE=40 timeout 300 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/tl/tl_$c.log 2>&1
grep "gbla timeline" gpurun_out/tl/tl_$c.log | tail -40 | head -60
done

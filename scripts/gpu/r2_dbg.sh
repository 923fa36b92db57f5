mkdir -p gpurun_out/dbg
for c in c0s c1 c3 c4 c2; do
if [ $c = c0s ]; then continue; fi
GBLA_BSUB_DEBUG=1 timeout 900 python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/dbg/d_$c.log 2>&1; grep "gbla echelon" gpurun_out/dbg/d_$c.log | head -2
done

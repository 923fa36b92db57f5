mkdir -p gpurun_out/c4g
for g in 0 16 32 64; do
GBLA_SWEEP_GROUP=$g timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c4g/c4_$g.log 2>&1; echo "c4 group $g rc=$?"
grep '^{' gpurun_out/c4g/c4_$g.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c4 group', '$g', d['ms_per_step'], d['kernel_ms_per_step'], d['clocks']['sm_mhz'])"
done

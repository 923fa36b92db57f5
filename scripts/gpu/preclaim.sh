# sweep pre-claim (GBLA_SWEEP_PRECLAIM): sweep-path parity tests, then c2/c1/c3 benches with it on and off
mkdir -p gpurun_out/pc
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "preclaim or backsub or c0_full or scaled or xt_batches or long_acc or c1_full or c3_full" > gpurun_out/pc/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pc/pytest.log
for c in c2 c1 c3; do for v in 1 0 1 0; do
GBLA_SWEEP_PRECLAIM=$v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pc/bench_${c}_$v.log 2>&1
echo "$c preclaim=$v rc=$? $(grep '^{' gpurun_out/pc/bench_${c}_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_step"], d["kernel_ms_per_step"], d["clocks"]["sm_mhz"])')"
done; done

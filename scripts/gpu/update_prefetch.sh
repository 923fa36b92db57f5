# K7' update with the D row segment read before the accumulator wait: update-path parity tests, c2/c3/c1 benches
mkdir -p gpurun_out/up
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "unfused or c0_full or scaled or xt_batches or long_acc or c1_full or sharded" > gpurun_out/up/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/up/pytest.log
for c in c2 c3 c1; do for r in 1 2; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/up/bench_${c}_$r.log 2>&1
echo "$c run$r rc=$? $(grep '^{' gpurun_out/up/bench_${c}_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_step"], d["kernel_ms_per_step"], d["clocks"]["sm_mhz"])')"
done; done

# K7' persistent tile walk (GBLA_UPD_PERSIST): update-path parity tests, c2/c3/c1 benches on / off
mkdir -p gpurun_out/ps
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "unfused or c0_full or scaled or xt_batches or long_acc or c1_full or c3_full or sharded or one_cta or edge or backsub_rref" > gpurun_out/ps/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ps/pytest.log
for c in c2 c3 c1; do for v in 1 0 1 0; do
GBLA_UPD_PERSIST=$v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ps/bench_${c}_$v.log 2>&1
echo "$c persist=$v rc=$? $(grep '^{' gpurun_out/ps/bench_${c}_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(d["ms_per_step"], d["kernel_ms_per_step"], d["clocks"]["sm_mhz"])')"
done; done

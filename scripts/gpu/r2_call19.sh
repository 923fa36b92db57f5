mkdir -p gpurun_out/r2c19
GBLA_K11_K128_PAIR=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "modgemm" > gpurun_out/r2c19/pytest_modgemm.log 2>&1; tail -2 gpurun_out/r2c19/pytest_modgemm.log
for pr in 0 1; do for pm in 0 1; do echo "k128 pair $pr perm $pm"; GBLA_K11_K128_PAIR=$pr GBLA_K11_BENCH_PERM=$pm timeout 120 python scripts/k11_bench.py 40000x45056x128 8192x45056x128 2048x20000x128; done; done > gpurun_out/r2c19/k11.log 2>&1
cat gpurun_out/r2c19/k11.log

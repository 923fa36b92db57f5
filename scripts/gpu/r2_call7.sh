mkdir -p gpurun_out/r2c7
for np in 64 128; do for e in 0 2; do echo "pair $np exp $e"; GBLA_K11_PAIR=$np GBLA_K11_EXP=$e timeout 120 python scripts/k11_bench.py 40000x45056x512 16384x16384x512; done; done > gpurun_out/r2c7/k11.log 2>&1
GBLA_K11_PAIR=128 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "modgemm" > gpurun_out/r2c7/pytest_modgemm.log 2>&1; tail -3 gpurun_out/r2c7/pytest_modgemm.log
cat gpurun_out/r2c7/k11.log

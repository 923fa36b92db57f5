mkdir -p gpurun_out/r2c5
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "modgemm" > gpurun_out/r2c5/pytest_modgemm.log 2>&1; tail -3 gpurun_out/r2c5/pytest_modgemm.log
for e in 0 2; do echo "pair exp $e"; GBLA_K11_EXP=$e timeout 120 python scripts/k11_bench.py 40000x45056x512 16384x16384x512; done > gpurun_out/r2c5/k11.log 2>&1
echo "single exp 0"  >> gpurun_out/r2c5/k11.log; GBLA_K11_PAIR=0 timeout 120 python scripts/k11_bench.py 40000x45056x512 >> gpurun_out/r2c5/k11.log 2>&1
cat gpurun_out/r2c5/k11.log

mkdir -p gpurun_out/r2c3
for e in 0 1 2; do echo "exp $e"; GBLA_K11_EXP=$e python scripts/k11_bench.py 40000x45056x512 40000x45056x128 16384x16384x512; done > gpurun_out/r2c3/k11_exp.log 2>&1
cat gpurun_out/r2c3/k11_exp.log

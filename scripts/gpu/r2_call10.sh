mkdir -p gpurun_out/r2c10
for e in 3 2 1 0; do echo "uv-alt exp $e"; GBLA_K11_EXP=$e timeout 120 python scripts/k11_bench.py 40000x45056x512 16384x16384x512; done > gpurun_out/r2c10/k11.log 2>&1
cat gpurun_out/r2c10/k11.log

mkdir -p gpurun_out/r2c14
for pm in 0 1; do echo "perm $pm"; GBLA_K11_BENCH_PERM=$pm timeout 120 python scripts/k11_bench.py 40000x45056x512 8192x45056x512 40000x45056x128; done > gpurun_out/r2c14/k11.log 2>&1
cat gpurun_out/r2c14/k11.log

mkdir -p gpurun_out/r2c31
for lib in "" variants/libgbla_nsb2.so; do
 for e in 0 1 2; do
  echo "lib=$lib exp=$e"
  GBLA_LIB=$lib GBLA_K11_EXP=$e timeout 120 python scripts/k11_bench.py 40000x45056x512 8192x90112x512
 done
done > gpurun_out/r2c31/k11.log 2>&1
cat gpurun_out/r2c31/k11.log

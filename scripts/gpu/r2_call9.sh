mkdir -p gpurun_out/r2c9
for e in 3 2; do echo "uv exp $e"; GBLA_K11_EXP=$e timeout 120 python scripts/k11_bench.py 16384x16384x512; done > gpurun_out/r2c9/k11.log 2>&1
cat gpurun_out/r2c9/k11.log
GBLA_K11_EXP=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modgemm_mk2 -s 1 -c 1 -o gpurun_out/r2c9/uv_exp2 python scripts/k11_bench.py 16384x16384x512 > gpurun_out/r2c9/ncu1.log 2>&1
GBLA_K11_EXP=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modgemm_mk2 -s 1 -c 1 -o gpurun_out/r2c9/uv_exp3 python scripts/k11_bench.py 16384x16384x512 > gpurun_out/r2c9/ncu2.log 2>&1
ls gpurun_out/r2c9

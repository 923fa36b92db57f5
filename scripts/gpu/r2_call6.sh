mkdir -p gpurun_out/r2c6
GBLA_K11_EXP=2 python scripts/k11_bench.py 16384x16384x512 > gpurun_out/r2c6/plain.log 2>&1 && \
GBLA_K11_EXP=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modgemm_mk2 -s 1 -c 1 -o gpurun_out/r2c6/mk2_exp2 python scripts/k11_bench.py 16384x16384x512 > gpurun_out/r2c6/ncu1.log 2>&1
GBLA_K11_PAIR=0 GBLA_K11_EXP=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modgemm_ws -s 1 -c 1 -o gpurun_out/r2c6/mk1_exp2 python scripts/k11_bench.py 16384x16384x512 > gpurun_out/r2c6/ncu2.log 2>&1
tail -2 gpurun_out/r2c6/ncu1.log gpurun_out/r2c6/ncu2.log

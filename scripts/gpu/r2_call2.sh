mkdir -p gpurun_out/r2c2
python -m pytest tests/test_gpu_parity.py -q -k modgemm > gpurun_out/r2c2/pytest_modgemm.log 2>&1; tail -3 gpurun_out/r2c2/pytest_modgemm.log
python scripts/k11_bench.py > gpurun_out/r2c2/k11.log 2>&1 && cat gpurun_out/r2c2/k11.log && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_modgemm_ws -s 1 -c 1 -o gpurun_out/r2c2/k11_mk python scripts/k11_bench.py 40000x45056x512 > gpurun_out/r2c2/ncu.log 2>&1
tail -2 gpurun_out/r2c2/ncu.log

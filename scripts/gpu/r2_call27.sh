mkdir -p gpurun_out/r2c27
python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c27/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_modgemm_mk2 -s 303 -c 2 -o gpurun_out/r2c27/mk2_insitu python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c27/ncu.log 2>&1
tail -2 gpurun_out/r2c27/ncu.log

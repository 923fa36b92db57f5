set -x
mkdir -p gpurun_out/r2c1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python scripts/peaks/int8_peak.py > gpurun_out/r2c1/int8_peak.json 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/peaks/imad_peak.cu -o /tmp/imad_peak && /tmp/imad_peak > gpurun_out/r2c1/imad_peak.json 2>&1
python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c1/bench_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_modgemm_ws<0, 8, 1, 1>' -s 40 -c 4 -o gpurun_out/r2c1/mk_c2 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c1/ncu.log 2>&1
tail -3 gpurun_out/r2c1/ncu.log

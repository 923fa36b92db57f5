mkdir -p gpurun_out/r2c18
python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c18/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c18/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c18/ncu.log 2>&1
python scripts/launch_summary.py gpurun_out/r2c18/launches_c2.csv 1 > gpurun_out/r2c18/summary.txt 2>&1; head -14 gpurun_out/r2c18/summary.txt

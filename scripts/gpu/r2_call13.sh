mkdir -p gpurun_out/r2c13
timeout 600 python bench.py --config c2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c13/bench_c2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2c13/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c13/ncu.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r2c13/bench_c2.log'):
    if l.startswith('{'):
        d = json.loads(l); print(d['ms_per_step'], d['step_ms'], d['phase_ms_steps'], d['kernel_ms_per_step'])
PY
python scripts/launch_summary.py gpurun_out/r2c13/launches_c2.csv 1 | head -20

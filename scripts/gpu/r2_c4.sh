mkdir -p gpurun_out/r2c4full
timeout 1200 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c4full/bench_c4.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r2c4full/bench_c4.log'):
    if l.startswith('{'):
        d = json.loads(l); print('c4', d['ms_per_step'], d['phase_ms'], d['kernel_ms_per_step'], d['clocks'])
PY
tail -3 gpurun_out/r2c4full/bench_c4.log

mkdir -p gpurun_out/r2c22
for c in c1 c2; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c22/bench_$c.log 2>&1; done
python - <<'PY'
import json
for c in ('c1','c2'):
    for l in open(f'gpurun_out/r2c22/bench_{c}.log'):
        if l.startswith('{'):
            d = json.loads(l); print(c, d['ms_per_step'], d['step_ms'], d['phase_ms'], d['kernel_ms_per_step'])
PY
timeout 300 python scripts/f2_time.py c1 > gpurun_out/r2c22/f2.log 2>&1; cat gpurun_out/r2c22/f2.log
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/r2c22/pytest.log 2>&1; tail -3 gpurun_out/r2c22/pytest.log

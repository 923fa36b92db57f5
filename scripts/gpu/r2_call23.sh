mkdir -p gpurun_out/r2c23
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/r2c23/pytest.log 2>&1; tail -3 gpurun_out/r2c23/pytest.log
for c in c1 c2 c3; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c23/bench_$c.log 2>&1; done
python - <<'PY'
import json
for c in ('c1','c2','c3'):
    for l in open(f'gpurun_out/r2c23/bench_{c}.log'):
        if l.startswith('{'):
            d = json.loads(l); print(c, d['ms_per_step'], d['phase_ms'], d['kernel_ms_per_step'])
PY

mkdir -p gpurun_out/r2c25
for r in 1 0; do GBLA_INT_RUNS=$r timeout 600 python bench.py --config c1 --flags 16 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c25/bench_int_runs$r.log 2>&1; done
python - <<'PY'
import json
for r in (1, 0):
    for l in open(f'gpurun_out/r2c25/bench_int_runs{r}.log'):
        if l.startswith('{'):
            d = json.loads(l); print('runs', r, d['ms_per_step'], d['phase_ms'])
PY
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "runs or int_pipe or engines" > gpurun_out/r2c25/pytest.log 2>&1; tail -2 gpurun_out/r2c25/pytest.log

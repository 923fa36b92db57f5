mkdir -p gpurun_out/r2c26
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "super_panels or runs or one_rank or full_rref" > gpurun_out/r2c26/pytest_quick.log 2>&1; tail -3 gpurun_out/r2c26/pytest_quick.log
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c26/bench_$c.log 2>&1; done
python - <<'PY'
import json
for c in ('c2','c3'):
    for l in open(f'gpurun_out/r2c26/bench_{c}.log'):
        if l.startswith('{'):
            d = json.loads(l); print(c, d['ms_per_step'], d['phase_ms'], d['kernel_ms_per_step'])
PY
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/r2c26/pytest.log 2>&1; tail -3 gpurun_out/r2c26/pytest.log

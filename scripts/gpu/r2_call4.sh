mkdir -p gpurun_out/r2c4
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "super_panels or modgemm or echelon_ref or scaled_configs" > gpurun_out/r2c4/pytest.log 2>&1; tail -5 gpurun_out/r2c4/pytest.log
timeout 600 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c4/bench_c2.log 2>&1; python - <<'PY'
import json
for l in open('gpurun_out/r2c4/bench_c2.log'):
    if l.startswith('{'):
        d = json.loads(l); print(d['ms_per_step'], d['phase_ms'], d['kernel_ms_per_step'], d['clocks'])
PY

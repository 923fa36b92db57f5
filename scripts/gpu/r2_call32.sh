mkdir -p gpurun_out/r2c32
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c0_full or c1_full or scaled_configs or echelon or super_panels or random_suite" > gpurun_out/r2c32/pytest.log 2>&1; tail -2 gpurun_out/r2c32/pytest.log
GBLA_PANEL_TRACE=1 timeout 300 python bench.py --config c1 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c32/trace_c1.log 2>&1; grep "panel2 trace" gpurun_out/r2c32/trace_c1.log | tail -1
timeout 300 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c32/bench_c1.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r2c32/bench_c1.log'):
    if l.startswith('{'):
        d = json.loads(l); print('c1', d['ms_per_step'], d['phase_ms'], d['kernel_ms_per_step'])
PY

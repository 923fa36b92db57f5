mkdir -p gpurun_out/r2c30
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "super_panels or c3_full" > gpurun_out/r2c30/pytest.log 2>&1; tail -2 gpurun_out/r2c30/pytest.log
timeout 600 python bench.py --config c2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c30/bench_c2.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r2c30/bench_c2.log'):
    if l.startswith('{'):
        d = json.loads(l); print('c2', d['ms_per_step'], d['phase_ms'], d['kernel_ms_per_step'], d['roofline']['frac'], d['roofline']['traffic'])
PY
GBLA_PANEL_TRACE=1 timeout 300 python bench.py --config c1 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c30/trace_c1.log 2>&1; grep "panel2 trace" gpurun_out/r2c30/trace_c1.log | tail -2
timeout 600 python scripts/wide_time.py c1 8388593 > gpurun_out/r2c30/wide_c1.log 2>&1; cat gpurun_out/r2c30/wide_c1.log

mkdir -p gpurun_out/r2c28
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "modgemm or super_panels or full_rref" > gpurun_out/r2c28/pytest.log 2>&1; tail -2 gpurun_out/r2c28/pytest.log
timeout 120 python scripts/k11_bench.py 40000x45056x512 16384x16384x512 > gpurun_out/r2c28/k11.log 2>&1; cat gpurun_out/r2c28/k11.log
timeout 600 python bench.py --config c2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c28/bench_c2.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r2c28/bench_c2.log'):
    if l.startswith('{'):
        d = json.loads(l); print('c2', d['ms_per_step'], d['phase_ms'], d['kernel_ms_per_step'])
PY

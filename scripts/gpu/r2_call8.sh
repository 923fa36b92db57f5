mkdir -p gpurun_out/r2c8
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "modgemm" > gpurun_out/r2c8/pytest_modgemm.log 2>&1; tail -3 gpurun_out/r2c8/pytest_modgemm.log
for e in 0 1 2; do echo "uv exp $e"; GBLA_K11_EXP=$e timeout 120 python scripts/k11_bench.py 40000x45056x512 16384x16384x512; done > gpurun_out/r2c8/k11.log 2>&1
cat gpurun_out/r2c8/k11.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "super_panels or echelon_ref or scaled_configs or xt_batches" > gpurun_out/r2c8/pytest.log 2>&1; tail -3 gpurun_out/r2c8/pytest.log
timeout 600 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c8/bench_c2.log 2>&1; python - <<'PY'
import json
for l in open('gpurun_out/r2c8/bench_c2.log'):
    if l.startswith('{'):
        d = json.loads(l); print(d['ms_per_step'], d['phase_ms'], d['kernel_ms_per_step'], d['clocks'])
PY

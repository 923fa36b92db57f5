mkdir -p gpurun_out/suite
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/suite/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/suite/pytest.log
for g in 0 32; do
GBLA_SWEEP_GROUP=$g timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/suite/c4_$g.log 2>&1
python - $g <<'PY'
import json,sys
for l in open(f'gpurun_out/suite/c4_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d = json.loads(l); print('c4 sweep group', sys.argv[1], d['ms_per_step'], d.get('phase_ms'), d.get('kernel_ms_per_step'))
PY
done

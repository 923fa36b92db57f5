mkdir -p gpurun_out/state
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/state/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/state/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/state/smoke.log 2>&1; echo "smoke rc=$?"
for c in c2 c1; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/state/bench_$c.log 2>&1
python - $c <<'PY'
import json,sys
for l in open(f'gpurun_out/state/bench_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], d['ms_per_step'], d.get('phase_ms'), d.get('kernel_ms_per_step'), d['roofline'], d.get('clocks'))
PY
done

mkdir -p gpurun_out/verify
timeout 1800 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/verify/pytest.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/verify/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/verify/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/verify/smoke.log
for c in c2 c1 c3 c4; do
st=3; [ $c = c4 ] && st=1
timeout 900 python bench.py --config $c --steps $st --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/verify/b_$c.log 2>&1
python - $c <<'PY'
import json,sys
for l in open(f'gpurun_out/verify/b_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], d['ms_per_step'], d.get('phase_ms'), d.get('kernel_ms_per_step'), d['e2e'], d['clocks'])
PY
done

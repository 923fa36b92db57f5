mkdir -p gpurun_out/f2
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/f2/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f2/smoke.log
timeout 900 python bench.py > gpurun_out/f2/bench_default.log 2>&1; echo "bench default rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/f2/bench_c2.log 2>&1; echo "bench c2 rc=$?"
for c in c1 c3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f2/bench_$c.log 2>&1; echo "bench $c rc=$?"; done
timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/f2/bench_c4.log 2>&1; echo "bench c4 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f2/bench_ref.log 2>&1; echo "ref rc=$?"
for c in default c1 c2 c3 c4 ref; do python - $c <<'PY'
import json,sys
for l in open(f'gpurun_out/f2/bench_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['ms_per_step'], d['value'], d.get('steps'), d.get('warmup'), d.get('kernel_ms_per_step'), d.get('clocks'))
PY
done

mkdir -p gpurun_out/sb
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/sb/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/sb/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sb/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/sb/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/sb/bench_c2.log 2>&1; echo "bench c2 rc=$?"
for c in c1 c3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sb/bench_$c.log 2>&1; echo "bench $c rc=$?"; done
timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sb/bench_c4.log 2>&1; echo "bench c4 rc=$?"
for c in c1 c2 c3 c4; do python - $c <<'PY'
import json,sys
for l in open(f'gpurun_out/sb/bench_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['ms_per_step'], d['value'], d['kernel_ms_per_step'], d['roofline']['frac'], d['clocks'])
PY
done

mkdir -p gpurun_out/sw2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c0_full or random or scaled or chunked or backsub or xt_batches or c1_full" > gpurun_out/sw2/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/sw2/pytest.log
for c in c2 c1 c3; do
timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sw2/b_$c.log 2>&1
python - $c <<'PY'
import json,sys
for l in open(f'gpurun_out/sw2/b_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], d['ms_per_step'], d.get('phase_ms'), d.get('kernel_ms_per_step'), {k: d['roofline'].get(k) for k in ('kernel','frac','executed_TOPS','executed_frac')})
PY
tail -2 gpurun_out/sw2/b_$c.log | grep -iv '^{' | cut -c1-300
done

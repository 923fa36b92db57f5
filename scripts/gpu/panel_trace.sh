mkdir -p gpurun_out/trace
for c in c1 c2; do
GBLA_PANEL_TRACE=1 timeout 300 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/trace/t_$c.log 2>&1; grep "panel2 trace" gpurun_out/trace/t_$c.log | tail -1
GBLA_ECH_TIMELINE=12 timeout 300 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/trace/tl_$c.log 2>&1; grep "gbla timeline" gpurun_out/trace/tl_$c.log | tail -12
timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/trace/b_$c.log 2>&1
python - $c <<'PY'
import json,sys
for l in open(f'gpurun_out/trace/b_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], d['ms_per_step'], d.get('phase_ms'), d.get('kernel_ms_per_step'))
PY
done

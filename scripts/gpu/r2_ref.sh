mkdir -p gpurun_out/ref
for c in c2 c1 c3; do
timeout 600 python bench.py --config $c --flags 128 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ref/ref_$c.log 2>&1
python - $c <<'PY'
import json,sys
for l in open(f'gpurun_out/ref/ref_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], 'REF', d['ms_per_step'], d.get('phase_ms'), d.get('kernel_ms_per_step'), d.get('rank_D'))
PY
done

mkdir -p gpurun_out/ref
for c in c2 c1; do
for env in "GBLA_SP=1 GBLA_NO_PREFIX_SLOTS=1" "GBLA_SP=1" "GBLA_NO_PREFIX_SLOTS=1"; do
env $env timeout 600 python bench.py --config $c --flags 128 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ref/ref2_$c.log 2>&1
python - $c "$env" <<'PY'
import json,sys
for l in open(f'gpurun_out/ref/ref2_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], sys.argv[2], 'REF', d['ms_per_step'], d.get('phase_ms'), d.get('kernel_ms_per_step'), d.get('rank_D'))
PY
done
done

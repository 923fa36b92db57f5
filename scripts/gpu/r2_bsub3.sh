mkdir -p gpurun_out/bsub
for g in auto 0 4 8 32 64; do
if [ $g = auto ]; then unset GBLA_BSUB_GROUP; else export GBLA_BSUB_GROUP=$g; fi
timeout 600 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bsub/g_$g.log 2>&1
python - $g <<'PY'
import json,sys
for l in open(f'gpurun_out/bsub/g_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d = json.loads(l); print('group', sys.argv[1], d['ms_per_step'], d.get('kernel_ms_per_step'), {k: d['roofline'].get(k) for k in ('kernel','frac','executed_TOPS','executed_frac','algorithmic_over_executed')})
PY
done
unset GBLA_BSUB_GROUP
for g in 0 4 8 64; do
GBLA_SWEEP_GROUP=$g timeout 600 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bsub/sg_$g.log 2>&1
python - $g <<'PY'
import json,sys
for l in open(f'gpurun_out/bsub/sg_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d = json.loads(l); print('sweep group', sys.argv[1], d['ms_per_step'], d.get('kernel_ms_per_step'))
PY
done

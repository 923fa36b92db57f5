mkdir -p gpurun_out/c4b
GBLA_BACKSUB=1 timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c4b/c4_b1.log 2>&1
python - <<'PY'
import json,sys
for l in open('gpurun_out/c4b/c4_b1.log'):
    if l.startswith('{'):
        d = json.loads(l); print('c4 bsub=1', d['ms_per_step'], d.get('phase_ms'), d.get('kernel_ms_per_step'))
PY
tail -2 gpurun_out/c4b/c4_b1.log | cut -c1-300
bash scripts/gpu/r2_ncu_sweep.sh

mkdir -p gpurun_out/rp4
for sfx in full pre; do
if [ $sfx = full ]; then export GBLA_REF_FULLSCAN=1; else unset GBLA_REF_FULLSCAN; fi
timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/rp4/c4_$sfx.log 2>&1; echo "c4 $sfx rc=$?"
timeout 600 python bench.py --config c2 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/rp4/c2_$sfx.log 2>&1; echo "c2 $sfx rc=$?"
done
for f in gpurun_out/rp4/*.log; do python - $f <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['ms_per_step'], d['phase_ms'], d['kernel_ms_per_step'], d['clocks']['sm_mhz'])
PY
done

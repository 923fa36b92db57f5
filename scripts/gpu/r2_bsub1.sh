mkdir -p gpurun_out/bsub
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c0_full or random or edge or scaled" > gpurun_out/bsub/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/bsub/pytest.log
for c in c2 c1 c3; do
for bs in 1 0; do
GBLA_BACKSUB=$bs timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bsub/b_${c}_$bs.log 2>&1
python - $c $bs <<'PY'
import json,sys
for l in open(f'gpurun_out/bsub/b_{sys.argv[1]}_{sys.argv[2]}.log'):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], 'bsub', sys.argv[2], d['ms_per_step'], d.get('phase_ms'), d.get('kernel_ms_per_step'), d.get('rank_D'))
PY
tail -3 gpurun_out/bsub/b_${c}_$bs.log | grep -v '^{' | head -3
done
done

mkdir -p gpurun_out/vf
timeout 1500 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/vf/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/vf/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/vf/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/vf/smoke.log
timeout 900 python bench.py > gpurun_out/vf/bench_default.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/vf/bench_default.log | cut -c1-400
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/vf/bench_c1.log 2>&1; echo "bench c1 rc=$?"; grep '^{' gpurun_out/vf/bench_c1.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/vf/bench_ref.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/vf/bench_ref.log | cut -c1-200

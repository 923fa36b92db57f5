#!/bin/bash
# final evidence (c1 only + GPU suite + launch list): the build with the B-tile prefetch
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/f_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/f_bench_c1.log 2>&1; echo "bench rc=$?" >> gpurun_out/f_bench_c1.log
timeout 300 python bench.py --flags 128 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/f_bench_c1_ref.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_bench_reference.log 2>&1
timeout 400 python bench.py --config c3 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/f_bench_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/f_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/f_ncu.log

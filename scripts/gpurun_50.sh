#!/bin/bash
# round-1 evidence for the current build: tests, bench, launch list with DRAM bytes, full capture of top kernels
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_all.log
timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_final.log
CMD="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain50.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_c1.csv $CMD > gpurun_out/ncu50a.log 2>&1 ; \
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:k_sweep|k_panel2|k_modgemm_ws' -s 6 -c 4 -o gpurun_out/prof50 $CMD > gpurun_out/ncu50b.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu50b.log

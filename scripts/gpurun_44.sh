#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python bench.py --config c2 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain44.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu44.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu44.log

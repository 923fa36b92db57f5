#!/bin/bash
# profiles: ncu full capture of k_sweep (c1); launch list of c2 (1 step) for the trailing-update breakdown
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep -c 1 -o gpurun_out/sweep_c1 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_sweep.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python bench.py --config c2 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain45.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k 'regex:k_modgemm_ws' -s 723 -c 1 -o gpurun_out/prof45 $CMD > gpurun_out/ncu45.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu45.log

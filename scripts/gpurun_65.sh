#!/bin/bash
# 8(f) f1: GBLA_ECHELON_REF parity + benches (c1, c3) next to the full RREF
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 2 --e2e-steps 0 --no-cpu-baseline --flags 128 > gpurun_out/b1_ref.log 2>&1
timeout 600 python bench.py --config c3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --flags 128 > gpurun_out/b3_ref.log 2>&1

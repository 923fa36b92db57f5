mkdir -p gpurun_out/r2c17
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "one_rank or errors or sharded" > gpurun_out/r2c17/pytest_nccl.log 2>&1; tail -15 gpurun_out/r2c17/pytest_nccl.log
timeout 600 python bench.py --steps 3 --warmup 2 --e2e-steps 1 --cpu-targets 64 > gpurun_out/r2c17/bench_c2.log 2>&1; tail -c 3000 gpurun_out/r2c17/bench_c2.log

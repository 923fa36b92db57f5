mkdir -p gpurun_out/r2c20
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_rref" > gpurun_out/r2c20/pytest.log 2>&1; tail -30 gpurun_out/r2c20/pytest.log

mkdir -p gpurun_out/r2c29
timeout 900 python -m pytest tests/test_gpu_wide.py -q -x > gpurun_out/r2c29/pytest.log 2>&1; tail -30 gpurun_out/r2c29/pytest.log

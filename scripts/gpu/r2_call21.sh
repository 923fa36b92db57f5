mkdir -p gpurun_out/r2c21
timeout 900 python -m pytest tests/test_gpu_formats.py -q -x > gpurun_out/r2c21/pytest.log 2>&1; tail -30 gpurun_out/r2c21/pytest.log
timeout 600 python scripts/format_bench.py c1 > gpurun_out/r2c21/fmt_c1.log 2>&1; cat gpurun_out/r2c21/fmt_c1.log
timeout 600 python scripts/f2_time.py c1 c3 > gpurun_out/r2c21/f2.log 2>&1; cat gpurun_out/r2c21/f2.log

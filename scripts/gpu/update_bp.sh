# standard-order Step 3 on the INT pipe (k_update_from_bp, targets-major grid): parity, then timing
mkdir -p gpurun_out/ubp
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bprime or standard_order or errors" > gpurun_out/ubp/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ubp/pytest.log
timeout 900 python scripts/trsm_time.py c1 c3 c2 --tc-only > gpurun_out/ubp/time_default.jsonl 2> gpurun_out/ubp/time_default.err; echo "time rc=$?"; cat gpurun_out/ubp/time_default.jsonl; tail -3 gpurun_out/ubp/time_default.err

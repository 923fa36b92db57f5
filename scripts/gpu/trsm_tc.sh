# tensor-core TRSM (gbla_reduce_B default): parity tests of the standard order, then timing
mkdir -p gpurun_out/trsm
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bprime or standard_order or errors or full_rref" > gpurun_out/trsm/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/trsm/pytest.log
timeout 900 python scripts/trsm_time.py c1 c3 > gpurun_out/trsm/time.jsonl 2> gpurun_out/trsm/time.err; echo "time rc=$?"; cat gpurun_out/trsm/time.jsonl; tail -3 gpurun_out/trsm/time.err
timeout 600 python scripts/trsm_time.py c2 --tc-only > gpurun_out/trsm/time_c2.jsonl 2> gpurun_out/trsm/time_c2.err; echo "time c2 rc=$?"; cat gpurun_out/trsm/time_c2.jsonl; tail -3 gpurun_out/trsm/time_c2.err

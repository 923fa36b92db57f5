# tensor-core TRSM (gbla_reduce_B default) and the K11 route of the standard-order update:
# parity tests of the standard order, then timing (INT engines: GBLA_TRSM_INT=1 / GBLA_UPDATE_BP=int)
mkdir -p gpurun_out/trsm
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bprime or standard_order or errors or full_rref" > gpurun_out/trsm/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/trsm/pytest.log
timeout 900 python scripts/trsm_time.py c1 c3 c2 --tc-only > gpurun_out/trsm/time_default.jsonl 2> gpurun_out/trsm/time_default.err; echo "time rc=$?"; cat gpurun_out/trsm/time_default.jsonl; tail -3 gpurun_out/trsm/time_default.err
GBLA_UPDATE_BP=int timeout 900 python scripts/trsm_time.py c1 c3 > gpurun_out/trsm/time_int.jsonl 2> gpurun_out/trsm/time_int.err; echo "time int rc=$?"; cat gpurun_out/trsm/time_int.jsonl; tail -3 gpurun_out/trsm/time_int.err
GBLA_UPDATE_BP=tc timeout 600 python scripts/trsm_time.py c2 --tc-only > gpurun_out/trsm/time_c2_tc.jsonl 2> gpurun_out/trsm/time_c2_tc.err; echo "time c2 tc rc=$?"; cat gpurun_out/trsm/time_c2_tc.jsonl; tail -3 gpurun_out/trsm/time_c2_tc.err

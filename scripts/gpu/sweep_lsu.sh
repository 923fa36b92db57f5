mkdir -p gpurun_out/lsu
GBLA_SWEEP_LSU=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c0_full or random_suite_new or scaled or c1_full or xt_batches or emulated or backsub_rref" > gpurun_out/lsu/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/lsu/pytest.log
ENV_SWEEP_STEPS=4 timeout 300 python scripts/env_sweep.py c1 "" "GBLA_SWEEP_LSU=1" > gpurun_out/lsu/c1.jsonl 2>gpurun_out/lsu/c1.err; cut -c1-200 gpurun_out/lsu/c1.jsonl
ENV_SWEEP_STEPS=2 timeout 600 python scripts/env_sweep.py c2 "" "GBLA_SWEEP_LSU=1" > gpurun_out/lsu/c2.jsonl 2>gpurun_out/lsu/c2.err; cut -c1-200 gpurun_out/lsu/c2.jsonl
tail -n 2 gpurun_out/lsu/*.err

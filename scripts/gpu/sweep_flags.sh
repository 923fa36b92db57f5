mkdir -p gpurun_out/sf
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c0_full or random_suite_new or scaled or long_acc or backsub or c1_full or c3_full or xt_batches or emulated" > gpurun_out/sf/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/sf/pytest.log
ENV_SWEEP_STEPS=4 timeout 300 python scripts/env_sweep.py c1 "" > gpurun_out/sf/c1.jsonl 2>gpurun_out/sf/c1.err; cut -c1-260 gpurun_out/sf/c1.jsonl
ENV_SWEEP_STEPS=2 timeout 600 python scripts/env_sweep.py c2 ""  > gpurun_out/sf/c2.jsonl 2>gpurun_out/sf/c2.err; cut -c1-260 gpurun_out/sf/c2.jsonl
ENV_SWEEP_STEPS=2 timeout 300 python scripts/env_sweep.py c3 "" > gpurun_out/sf/c3.jsonl 2>gpurun_out/sf/c3.err; cut -c1-260 gpurun_out/sf/c3.jsonl
tail -n 2 gpurun_out/sf/*.err

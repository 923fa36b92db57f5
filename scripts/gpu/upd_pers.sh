mkdir -p gpurun_out/up2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "prefix or random_suite_new or scaled or unfused or c0_full or c1_full or xt_batches or long_acc or emulated or full_rref or c3_full or one_rank" > gpurun_out/up2/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/up2/pytest.log
ENV_SWEEP_STEPS=4 timeout 300 python scripts/env_sweep.py c1 "GBLA_UPD_PERSIST=0" "" > gpurun_out/up2/c1.jsonl 2>gpurun_out/up2/c1.err; cut -c1-230 gpurun_out/up2/c1.jsonl
ENV_SWEEP_STEPS=2 timeout 600 python scripts/env_sweep.py c2 "GBLA_UPD_PERSIST=0" "" "GBLA_UPD_PERSIST=0" "" > gpurun_out/up2/c2.jsonl 2>gpurun_out/up2/c2.err; cut -c1-230 gpurun_out/up2/c2.jsonl
ENV_SWEEP_STEPS=2 timeout 300 python scripts/env_sweep.py c3 "GBLA_UPD_PERSIST=0" "" > gpurun_out/up2/c3.jsonl 2>gpurun_out/up2/c3.err; cut -c1-230 gpurun_out/up2/c3.jsonl
tail -n 2 gpurun_out/up2/*.err

mkdir -p gpurun_out/rp
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "backsub or echelon_ref or c1_full or c0_full or scaled or random_suite_new or one_rank or emulated or super_panels" > gpurun_out/rp/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/rp/pytest.log
ENV_SWEEP_STEPS=4 timeout 300 python scripts/env_sweep.py c1 "GBLA_REF_FULLSCAN=1" "" > gpurun_out/rp/c1.jsonl 2>gpurun_out/rp/c1.err; cut -c1-330 gpurun_out/rp/c1.jsonl
ENV_SWEEP_STEPS=2 timeout 600 python scripts/env_sweep.py c2 "GBLA_REF_FULLSCAN=1" "" > gpurun_out/rp/c2.jsonl 2>gpurun_out/rp/c2.err; cut -c1-330 gpurun_out/rp/c2.jsonl
tail -n 2 gpurun_out/rp/*.err

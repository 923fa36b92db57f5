mkdir -p gpurun_out/dist
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dist/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/dist/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "one_rank or emulated or echelon_ref_mode or xt_batches or c1_full" > gpurun_out/dist/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/dist/pytest.log

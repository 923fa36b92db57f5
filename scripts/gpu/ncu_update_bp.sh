# ncu --set full of the standard-order Step 3 INT kernel (k_update_from_bp) on c1
mkdir -p gpurun_out/ubp
GBLA_UPDATE_BP=int timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_update_from_bp -c 1 -o gpurun_out/ubp/ncu_update_bp_c1 python scripts/trsm_time.py c1 --tc-only > gpurun_out/ubp/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ubp/ncu.log

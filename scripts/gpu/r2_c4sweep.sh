mkdir -p gpurun_out/r2c4sw
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_sweep -c 2 --csv --log-file gpurun_out/r2c4sw/sweep_c4.csv python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2c4sw/ncu.log 2>&1
tail -3 gpurun_out/r2c4sw/ncu.log

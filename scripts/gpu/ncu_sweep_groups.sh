mkdir -p gpurun_out/grp
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,l1tex__m_xbar2l1tex_read_bytes.sum
for g in 0 16; do
GBLA_SWEEP_GROUP=$g timeout 900 ncu --metrics $M --clock-control none -k regex:"k_sweep|k_update_tc" -c 2 --csv python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/grp/ncu_c2_g$g.csv 2> gpurun_out/grp/ncu_c2_g$g.err
grep -E "dram__bytes_read|lts__t_sector_hit|tensor_cycles|gpu__time" gpurun_out/grp/ncu_c2_g$g.csv | awk -F'","' '{print $5, $13, $15}' | cut -c1-160
done
ENV_SWEEP_STEPS=1 timeout 1500 python scripts/env_sweep.py c4 "" "GBLA_SWEEP_GROUP=8" "GBLA_SWEEP_GROUP=16" "GBLA_SWEEP_GROUP=4" > gpurun_out/grp/c4.jsonl 2>gpurun_out/grp/c4.err; cat gpurun_out/grp/c4.jsonl; tail -n 3 gpurun_out/grp/c4.err

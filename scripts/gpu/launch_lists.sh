mkdir -p gpurun_out/r2lists
for c in c1 c2; do
python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2lists/plain_$c.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2lists/launches_$c.csv python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r2lists/ncu_$c.log 2>&1
python scripts/launch_summary.py gpurun_out/r2lists/launches_$c.csv 1 > gpurun_out/r2lists/summary_$c.txt 2>&1
done
head -12 gpurun_out/r2lists/summary_c2.txt

# launch lists (ncu, per-kernel device time + DRAM bytes) of one bench step, c1 and c2, after the
# plain run of the same command exits 0
mkdir -p gpurun_out/ll
for c in c1 c2; do
timeout 600 python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ll/plain_$c.log 2>&1; echo "plain $c rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll/launches_$c.csv python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ll/ncu_$c.log 2>&1; echo "list $c rc=$?"
python scripts/launch_summary.py gpurun_out/ll/launches_$c.csv 1 > gpurun_out/ll/launches_${c}_summary.txt 2>&1; head -10 gpurun_out/ll/launches_${c}_summary.txt
done

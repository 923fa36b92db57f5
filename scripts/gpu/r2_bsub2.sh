mkdir -p gpurun_out/bsub
python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/bsub/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bsub/ncu_c2.log 2>&1
python scripts/launch_summary.py gpurun_out/bsub/launches_c2.csv 1 > gpurun_out/bsub/summary_c2.txt 2>&1
head -30 gpurun_out/bsub/summary_c2.txt

# round-end evidence: GPU suite, smoke, bench lines (c2 headline + c1/c3/c4), launch lists with DRAM
# bytes (c1, c2), one ncu --set full capture of the c2 sparse sweep
mkdir -p gpurun_out/fin
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/fin/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/fin/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fin/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/fin/bench_c2.log 2>&1; echo "bench c2 rc=$?"; grep '^{' gpurun_out/fin/bench_c2.log | cut -c1-200
for c in c1 c3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fin/bench_$c.log 2>&1; echo "bench $c rc=$?"; done
timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/fin/bench_c4.log 2>&1; echo "bench c4 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin/bench_ref.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/fin/bench_ref.log | cut -c1-200
for c in c1 c2; do
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fin/launches_$c.csv python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fin/ncu_list_$c.log 2>&1; echo "list $c rc=$?"
python scripts/launch_summary.py gpurun_out/fin/launches_$c.csv 1 > gpurun_out/fin/launches_${c}_summary.txt 2>&1; head -12 gpurun_out/fin/launches_${c}_summary.txt
done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_sweep -c 1 -o gpurun_out/fin/ncu_sweep_c2 python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fin/ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -2 gpurun_out/fin/ncu_full.log

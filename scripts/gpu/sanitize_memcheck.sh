mkdir -p gpurun_out/san
timeout 1500 compute-sanitizer --tool memcheck --log-file gpurun_out/san/memcheck.txt python scripts/sanitize_run.py > gpurun_out/san/memcheck_stdout.txt 2>&1; echo "rc=$?"
tail -5 gpurun_out/san/memcheck.txt; tail -3 gpurun_out/san/memcheck_stdout.txt

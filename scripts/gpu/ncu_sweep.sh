mkdir -p gpurun_out/ncusw
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_sweep -c 2 -o gpurun_out/ncusw/sweep_c2 python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncusw/ncu.log 2>&1
tail -3 gpurun_out/ncusw/ncu.log

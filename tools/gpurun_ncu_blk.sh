mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blk_ -s 4 -c 4 -o gpurun_out/prof_blk python bench.py --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_blk.log 2>&1; tail -1 gpurun_out/ncu_blk.log

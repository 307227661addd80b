mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_blk_rhs|k_blk_gather" -s 2 -c 2 -o gpurun_out/prof_mom python bench.py --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs > gpurun_out/ncu_mom.log 2>&1; tail -1 gpurun_out/ncu_mom.log

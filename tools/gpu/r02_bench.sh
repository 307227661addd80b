# round 2: C5 headline bench (both arms), 2-rank functional run of the
# strong-scaling path (gloo, one GPU), C5 launch list + ncu of the step kernels
mkdir -p gpurun_out
free -g > gpurun_out/host_mem.txt; nproc >> gpurun_out/host_mem.txt
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json | head -c 3000; echo; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; cat gpurun_out/bench_ref.json | head -c 600; echo
FPB_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; head -c 1500 gpurun_out/bench_n2.json; echo; tail -3 gpurun_out/bench_n2.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows_pairs|k_blk_rhs|k_blk_gather" -s 6 -c 3 -o gpurun_out/prof_c5 python bench.py --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log

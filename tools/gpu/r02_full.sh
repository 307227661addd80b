# round 2 checkpoint: full GPU suite, smoke, both bench arms, launch list and ncu of the step kernels
mkdir -p gpurun_out
free -g > gpurun_out/host_mem.txt; nproc >> gpurun_out/host_mem.txt
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; head -c 1500 gpurun_out/bench.json; echo; tail -2 gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; head -c 400 gpurun_out/bench_ref.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows_pairs|k_blk_rhs|k_blk_gather" -s 8 -c 4 -o gpurun_out/prof_c5 python bench.py --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hex" -s 3 -c 3 -o gpurun_out/prof_c4hex python tools/hexprobe.py --reps 1 > gpurun_out/ncu_hex.log 2>&1; tail -1 gpurun_out/ncu_hex.log

mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_auto.json 2> gpurun_out/bench.err; cat gpurun_out/bench_auto.json; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --scatter atomic > gpurun_out/bench_atomic.json 2>> gpurun_out/bench.err; cat gpurun_out/bench_atomic.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rows -s 4 -c 2 -o gpurun_out/prof_rows python bench.py --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_rows.log 2>&1; tail -2 gpurun_out/ncu_rows.log

mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "assembly" > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/kbench.py > gpurun_out/kbench.json 2>&1; cat gpurun_out/kbench.json
timeout 300 python tools/kbench.py --etype HEX08 --nx 60 --ny 60 --nz 60 --scatters atomic > gpurun_out/kbench_hex.json 2>&1; cat gpurun_out/kbench_hex.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rows -s 6 -c 2 -o gpurun_out/prof_rows2 python bench.py --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_rows.log 2>&1; tail -1 gpurun_out/ncu_rows.log

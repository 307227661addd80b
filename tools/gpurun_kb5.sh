mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/kbench.py --scatters auto > gpurun_out/kb_tet.json 2>&1; cat gpurun_out/kb_tet.json | tr -d '\n '; echo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rows" -s 2 -c 1 -o gpurun_out/prof_rows python bench.py --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 --no-solver > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log

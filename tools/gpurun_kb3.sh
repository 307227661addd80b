mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/kbench.py --scatters auto 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: v['ms'] for k, v in d.items() if isinstance(v, dict)})"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rows|k_blk_rhs" -s 4 -c 2 -o gpurun_out/prof_v4 python bench.py --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log

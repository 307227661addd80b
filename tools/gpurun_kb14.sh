mkdir -p gpurun_out
q() { python -c "import json,sys; d=json.load(sys.stdin); print({k.split('/')[1]: v['ms'] for k, v in d.items() if isinstance(v, dict)})"; }
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
echo "== rings"; timeout 300 python tools/kbench.py --scatters auto 2>&1 | q
echo "== no rings"; FPB_RINGS=0 timeout 300 python tools/kbench.py --scatters auto 2>&1 | q
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gradient_rings" -s 2 -c 1 -o gpurun_out/prof_rings python bench.py --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log

mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
echo "== hex 272^3"; timeout 600 python tools/kbench.py --scatters auto --etype HEX08 --nx 272 --ny 272 --nz 272 --reps 5 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: v['ms'] for k, v in d.items() if isinstance(v, dict)})"

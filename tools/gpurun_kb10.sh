mkdir -p gpurun_out
q() { python -c "import json,sys; d=json.load(sys.stdin); print({k.split('/')[1]: v['ms'] for k, v in d.items() if isinstance(v, dict)})"; }
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
echo "== hex 272^3"; timeout 600 python tools/kbench.py --scatters auto,atomic --etype HEX08 --nx 272 --ny 272 --nz 272 --reps 5 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: v['ms'] for k, v in d.items() if isinstance(v, dict)})"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rows_gl" -c 1 -o gpurun_out/prof_gl python tools/kbench.py --scatters auto --etype HEX08 --nx 96 --ny 96 --nz 96 --reps 1 > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log

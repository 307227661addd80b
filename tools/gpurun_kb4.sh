mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/kbench.py --scatters auto > gpurun_out/kb_tet.json 2>&1; cat gpurun_out/kb_tet.json | tr -d '\n '; echo
timeout 600 python tools/kbench.py --scatters auto --etype HEX08 --nx 272 --ny 272 --nz 272 --reps 5 > gpurun_out/kb_hex.json 2>&1; cat gpurun_out/kb_hex.json | tr -d '\n '; echo

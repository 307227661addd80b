# default build (TMA double-buffered output, 1-warp CTAs): parity, sanitizer, bench, ncu of the lines kernel
timeout 1200 python -m pytest tests/test_gpu_kuhn.py tests/test_gpu_scale.py tests/test_distributed_solver.py tests/test_gpu_assembly.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -k "gradients or aniso" -p no:cacheprovider 2>&1 | tail -1
timeout 600 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -k "gradients_match" -p no:cacheprovider 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['kernels_ms'])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_kuhn_grad_march" -s 2 -c 1 -o gpurun_out/kgtma2 python bench.py --steps 1 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs > gpurun_out/kgtma2.log 2>&1; tail -1 gpurun_out/kgtma2.log

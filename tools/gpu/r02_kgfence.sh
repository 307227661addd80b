# B_xyz lines with the all-lanes proxy fence: parity + timing
timeout 900 python -m pytest tests/test_gpu_kuhn.py tests/test_gpu_scale.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['kernels_ms'])"; done
timeout 600 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_kuhn.py -q -m gpu -k "gradients_match" -p no:cacheprovider 2>&1 | tail -1

# default build: Kuhn / scale / slab / hex parity, C5 bench (2 runs) + C3/C4 configs
timeout 1500 python -m pytest tests/test_gpu_kuhn.py tests/test_gpu_scale.py tests/test_distributed_solver.py tests/test_gpu_assembly.py tests/test_gpu_distorted.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['kernels_ms'])"; done
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-solver > gpurun_out/bench_cfg.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_cfg.json'));c=d['configs']
print({k:(v.get('ms_per_step') if isinstance(v,dict) else v) for k,v in c.items()})"

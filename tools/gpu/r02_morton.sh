mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_distorted.py tests/test_gpu_scale.py tests/test_distributed_solver.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_m.log 2>&1; tail -2 gpurun_out/pytest_m.log
for M in 0 1; do FPB_BLOCK_MORTON=$M timeout 900 python bench.py --steps 10 --warmup 3 --no-solver --no-cpu-baseline --e2e-steps 2 --soak 0 > gpurun_out/bench_m$M.json 2> gpurun_out/bench_m$M.err; python -c "
import json;d=json.load(open('gpurun_out/bench_m$M.json'));c=d['configs']
print('morton $M', d['value'],d['ms_per_step'],d['kernels_ms'], 'e2e', d['e2e']['value'], 'c2', c['c2']['kernels_ms'], 'c3', c['c3']['ms_per_step'], 'c4', c['c4']['ms_per_step'], {k:v['ms'] for k,v in c['c4']['kernels'].items()}, 'c4e2e', c['c4']['e2e']['value'])"; tail -1 gpurun_out/bench_m$M.err; done

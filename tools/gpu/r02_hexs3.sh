mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_distorted.py tests/test_gpu_scale.py -q -m gpu -p no:cacheprovider -x -k "scalar or c4 or hex" > gpurun_out/pytest_s3.log 2>&1; tail -2 gpurun_out/pytest_s3.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-solver --no-cpu-baseline --e2e-steps 0 --soak 0 > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err; python -c "
import json;d=json.load(open('gpurun_out/bench_s3.json'));c=d['configs']
print(d['value'], 'c3', c['c3']['ms_per_step'], 'c4', c['c4']['ms_per_step'], {k:v['ms'] for k,v in c['c4']['kernels'].items()})"; tail -1 gpurun_out/bench_s3.err

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_scale.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_nbr.log 2>&1; tail -2 gpurun_out/pytest_nbr.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-solver --no-configs --no-cpu-baseline --e2e-steps 0 --soak 0 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; python -c "import json;d=json.load(open('gpurun_out/bench_quick.json'));print(d['value'],d['ms_per_step'],d['kernels_ms'],d['gpu_launches'])"; tail -2 gpurun_out/bench_quick.err

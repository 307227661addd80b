mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_distorted.py tests/test_gpu_scale.py tests/test_flow.py tests/test_reference_suite.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_kb.log 2>&1; tail -2 gpurun_out/pytest_kb.log
for v in default nokb; do
  if [ $v = kb2 ]; then export FPB_LIB_PATH=build_variants/kb2/libfempack_b200.so; else unset FPB_LIB_PATH; fi
  if [ $v = nokb ]; then export FPB_KUHN_BLOCKS=0; else unset FPB_KUHN_BLOCKS; fi
  timeout 900 python bench.py --steps 10 --warmup 3 --no-solver --no-cpu-baseline --e2e-steps 0 --soak 0 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; python -c "
import json;d=json.load(open('gpurun_out/bench_$v.json'));c=d['configs']
print('$v', d['value'],d['ms_per_step'],d['kernels_ms'], 'c2', c['c2']['kernels_ms'], 'c3', c['c3']['ms_per_step'])"; tail -1 gpurun_out/bench_$v.err
done

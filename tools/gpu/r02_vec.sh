mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_assembly.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_vec.log 2>&1; tail -1 gpurun_out/pytest_vec.log
for v in vec novec; do
  if [ $v = novec ]; then export FPB_LIB_PATH=build_variants/novec/libfempack_b200.so; else unset FPB_LIB_PATH; fi
  for rep in 1 2; do timeout 900 python bench.py --steps 20 --warmup 3 --no-solver --no-configs --no-cpu-baseline --e2e-steps 0 --soak 0 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; python -c "
import json;d=json.load(open('gpurun_out/bench_$v.json'));print('$v', d['value'],d['kernels_ms'])"; done
done

# Kuhn boundary-row kernel occupancy variants; build them first:
#   for m in 2 3; do bash tools/build_variant.sh bminb$m -DFPB_KGRAD_BMINB=$m; mkdir -p vtmp/b$m; cp build_variants/bminb$m/libfempack_b200.so vtmp/b$m/; done
mkdir -p gpurun_out
for v in default b2 b3; do
  if [ $v = default ]; then unset FPB_LIB_PATH; else export FPB_LIB_PATH=$PWD/vtmp/$v/libfempack_b200.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_kuhn_grad" --csv --log-file gpurun_out/bnd_$v.csv python bench.py --steps 2 --warmup 3 --soak 0 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs > gpurun_out/bnd_$v.log 2>&1
  echo "== $v"; grep -h "k_kuhn_grad_boundary" gpurun_out/bnd_$v.csv | awk -F'","' '{print $(NF-2), $NF}' | tail -6
done
unset FPB_LIB_PATH
timeout 600 python -m pytest tests/test_gpu_kuhn.py tests/test_gpu_scale.py -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 600 python bench.py --no-configs --no-solver --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_b.json'));print(d['ms_per_step'],d['kernels_ms'])"

# Kuhn momentum kernel: tests, timings of the default and the build_variants, ncu of the kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_kuhn.log 2>&1; tail -3 gpurun_out/pytest_kuhn.log
echo "== default"; timeout 600 python tools/kmom_probe.py --kchunks 0,32 --blocks 0 2>&1 | tail -4
for v in build_variants/*/; do
  echo "== $v"; FPB_LIB_PATH=$v/libfempack_b200.so timeout 600 python tools/kmom_probe.py --blocks 0 --kchunks 0,32 2>&1 | tail -4
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_kuhn_mom" -s 3 -c 1 -o gpurun_out/prof_kmom python tools/kmom_probe.py --sizes 256x256x256 --reps 1 --blocks 0 > gpurun_out/ncu_kmom.log 2>&1; tail -1 gpurun_out/ncu_kmom.log

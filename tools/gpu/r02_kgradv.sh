echo "== default"; timeout 600 python tools/kmom_probe.py --kchunks 0 --blocks 0 --grad 1 --sizes 256x256x256 2>&1 | grep grad_box
for v in build_variants/*/; do
  echo "== $v"; FPB_LIB_PATH=$v/libfempack_b200.so timeout 600 python tools/kmom_probe.py --kchunks 0 --blocks 0 --grad 1 --sizes 256x256x256 2>&1 | grep grad_box
done

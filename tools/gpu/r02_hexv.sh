echo "== default"; timeout 600 python tools/hexprobe.py --reps 5 2>&1 | tail -1
echo "== default canon64"; timeout 600 python tools/hexprobe.py --reps 5 --canon-rows 64 2>&1 | tail -1
for v in build_variants/*/; do
  echo "== $v"; FPB_LIB_PATH=$v/libfempack_b200.so timeout 600 python tools/hexprobe.py --reps 5 2>&1 | tail -1
done

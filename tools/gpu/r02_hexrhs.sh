K="--etype HEX08 --nx 272 --ny 272 --nz 272 --reps 5 --scatters auto"
Q() { python -c "import json,sys; d=json.load(sys.stdin); print({k.split('/')[1]: v['ms'] for k, v in d.items() if isinstance(v, dict) and 'rhs' in k})"; }
echo "== default"; timeout 900 python tools/kbench.py $K 2>&1 | Q
for v in build_variants/*/; do
  echo "== $v"; FPB_LIB_PATH=$v/libfempack_b200.so timeout 900 python tools/kbench.py $K 2>&1 | Q
done

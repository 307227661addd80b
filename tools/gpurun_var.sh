mkdir -p gpurun_out
for d in build_variants/*/; do
  echo "== $d"
  FPB_LIB_PATH=$d/libfempack_b200.so timeout 300 python tools/kbench.py --scatters auto 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: v['ms'] for k, v in d.items() if isinstance(v, dict) and 'rhs' in k})"
done

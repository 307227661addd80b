# variants first: t0 -DFPB_HEXR_TMA=0 (restructured loop, plain stores), t1 -DFPB_HEXR_TMA=1, orig (previous commit); copy to vtmp/<name>/
# HEX08 box row pass: TMA bulk stores of the staged CSR blocks (C4 B_xyz)
FPB_LIB_PATH=$PWD/vtmp/t1/libfempack_b200.so timeout 900 python -m pytest tests -q -m gpu -k "hex" -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do
for v in orig t0 t1; do
  echo "== $v"; FPB_LIB_PATH=$PWD/vtmp/$v/libfempack_b200.so timeout 600 python tools/hexprobe.py --reps 7 2>&1 | tail -1 | grep -o '"once_ms.*'
done
done

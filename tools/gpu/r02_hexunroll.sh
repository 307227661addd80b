# variants first: for u in 1 2; do bash tools/build_variant.sh u$u -DFPB_HEX_GUNROLL=$u; mkdir -p vtmp/u$u; cp build_variants/u$u/libfempack_b200.so vtmp/u$u/; done
# HEX08 Gauss-loop unroll (hex_rhs_integrate) vs the hex-box pencils' register spills: config-4 RHS timings
echo "== default (unroll 8)"; timeout 600 python tools/hexbox_probe.py --reps 5 2>&1 | tail -3
for v in u1 u2; do
  echo "== $v"; FPB_LIB_PATH=$PWD/vtmp/$v/libfempack_b200.so timeout 600 python tools/hexbox_probe.py --reps 5 2>&1 | tail -3
done

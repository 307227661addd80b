# variants first: for m in 4 12 15 3; do bash tools/build_variant.sh m$m -DFPB_HEXR_PFM=$m; mkdir -p vtmp/m$m; cp build_variants/m$m/libfempack_b200.so vtmp/m$m/; done
#   (vtmp/ travels to the GPU box; build_variants/ is gpurun-ignored)
# L2-prefetch distance sweep for the HEX08 box row pass (C4 B_xyz)
for rep in 1 2; do
echo "== default"; timeout 600 python tools/hexprobe.py --reps 7 2>&1 | tail -1 | grep -o '"once_ms.*'
for v in m4 m12 m15 m3; do
  echo "== $v"; FPB_LIB_PATH=$PWD/vtmp/$v/libfempack_b200.so timeout 600 python tools/hexprobe.py --reps 7 2>&1 | tail -1 | grep -o '"once_ms.*'
done
done

# variants first: for r in 192 184 176; do bash tools/build_variant.sh r$r -DFPB_KMOM_MAXNREG=$r; mkdir -p vtmp/r$r; cp build_variants/r$r/libfempack_b200.so vtmp/r$r/; done
# Kuhn momentum register cap (__maxnreg__) vs co-residency with the B_xyz lines kernel in the two-stream step
for rep in 1 2; do
echo "== default"; timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['kernels_ms'])"
for v in r192 r184 r176; do
echo "== $v"; FPB_LIB_PATH=$PWD/vtmp/$v/libfempack_b200.so timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['kernels_ms'])"
done
done

# variants first: tools/build_variant.sh ty10 -DFPB_KMOM_TY=10 -DFPB_KMOM_MAXNREG=200; ty9 (9, 224); ty12 (12, 168); copy to vtmp/<name>/
# Kuhn momentum: warps (cell rows) per CTA at the register cap that keeps one CTA per SM.  Result (not kept): TY 12 momentum 1.62 ms vs 1.56 at TY 8;
# TY 9 / 10 variants could not launch the other kinds (255 registers x 288 / 320 threads > 64 K), so their tests failed; TY stays 8.
FPB_LIB_PATH=$PWD/vtmp/ty10/libfempack_b200.so timeout 900 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -k "momentum" -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do
echo "== default (TY 8)"; timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['kernels_ms'])"
for v in ty9 ty10 ty12; do
echo "== $v"; FPB_LIB_PATH=$PWD/vtmp/$v/libfempack_b200.so timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['kernels_ms'])"
done
done

# variants first (tools/build_variant.sh): tma0 -DFPB_KGRAD_TMA=0; tma2 -DFPB_KGRAD_TMA=2 -DFPB_KGRAD_MINB=3;
#   tma2w1 -DFPB_KGRAD_TMA=2 -DFPB_KGRAD_WARPS=1 -DFPB_KGRAD_MINB=6; copy each libfempack_b200.so to vtmp/<name>/
# Kuhn B_xyz lines: TMA bulk stores of the staged CSR blocks vs plain coalesced stores
FPB_LIB_PATH=$PWD/vtmp/tma2/libfempack_b200.so timeout 900 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -k "gradients or ns_d or aniso" -p no:cacheprovider 2>&1 | tail -1
FPB_LIB_PATH=$PWD/vtmp/tma2w1/libfempack_b200.so timeout 900 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -k "gradients or ns_d or aniso" -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do
for v in tma0 tma2 tma2w1; do
echo "== $v"; FPB_LIB_PATH=$PWD/vtmp/$v/libfempack_b200.so timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-solver --no-configs 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'], d['kernels_ms'])"
done
done

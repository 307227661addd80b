timeout 900 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_distorted.py -q -m gpu -p no:cacheprovider -k "rhs or momentum" 2>&1 | tail -1
echo "== default"; FPB_KUHN_MOM=0 python tools/kmom_probe.py --kchunks 0 --blocks 0 --reps 10 | grep kuhn
echo "== old"; FPB_LIB_PATH=build_variants/blk_old/libfempack_b200.so FPB_KUHN_MOM=0 python tools/kmom_probe.py --kchunks 0 --blocks 0 --reps 10 | grep kuhn

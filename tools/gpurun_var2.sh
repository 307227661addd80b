q() { python -c "import json,sys; d=json.load(sys.stdin); print({k.split('/')[1]: v['ms'] for k, v in d.items() if isinstance(v, dict)})"; }
echo "== ld256 + inc/conn"; timeout 300 python tools/kbench.py --scatters auto 2>&1 | q
echo "== ld256 + inline"; FPB_ROWS_INLINE=1 timeout 300 python tools/kbench.py --scatters auto 2>&1 | q
echo "== ld64 + inc/conn"; FPB_LIB_PATH=build_variants/ld64/libfempack_b200.so timeout 300 python tools/kbench.py --scatters auto 2>&1 | q
echo "== ld64 + inline"; FPB_ROWS_INLINE=1 FPB_LIB_PATH=build_variants/ld64/libfempack_b200.so timeout 300 python tools/kbench.py --scatters auto 2>&1 | q

q() { python -c "import json,sys; d=json.load(sys.stdin); print({k.split('/')[1]: v['ms'] for k, v in d.items() if isinstance(v, dict)})"; }
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider 2>&1 | tail -1
echo "== pipelined"; timeout 300 python tools/kbench.py --scatters auto 2>&1 | q
for v in build_variants/*/; do echo "== $v"; FPB_LIB_PATH=$v/libfempack_b200.so timeout 300 python tools/kbench.py --scatters auto 2>&1 | q; done

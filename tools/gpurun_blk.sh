Q() { python -c "import json,sys; d=json.load(sys.stdin); print({k.split('/')[1]: v['ms'] for k, v in d.items() if isinstance(v, dict)})"; }
echo "== default"; timeout 300 python tools/kbench.py --scatters auto 2>&1 | Q
for v in build_variants/*/; do echo "== $v"; FPB_LIB_PATH=$v/libfempack_b200.so timeout 300 python tools/kbench.py --scatters auto 2>&1 | Q; done
echo "== default again"; timeout 300 python tools/kbench.py --scatters auto 2>&1 | Q

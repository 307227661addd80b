Q() { python -c "import json,sys; d=json.load(sys.stdin); print({k.split('/')[1]: v['ms'] for k, v in d.items() if isinstance(v, dict)})"; }
H="--scatters auto --etype HEX08 --nx 272 --ny 272 --nz 272 --reps 5"
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider 2>&1 | tail -2
echo "== new"; timeout 600 python tools/kbench.py $H 2>&1 | Q
for v in build_variants/*/; do echo "== $v"; FPB_LIB_PATH=$v/libfempack_b200.so timeout 600 python tools/kbench.py $H 2>&1 | Q; done

timeout 900 python -m pytest tests/test_gpu_kuhn.py -q -m gpu -p no:cacheprovider -k "hex" 2>&1 | tail -2
K="--etype HEX08 --nx 272 --ny 272 --nz 272 --reps 5 --scatters auto"
Q() { python -c "import json,sys; d=json.load(sys.stdin); print({k.split('/')[1]: v['ms'] for k, v in d.items() if isinstance(v, dict) and 'rhs' in k})"; }
echo "== pencils"; timeout 900 python tools/kbench.py $K 2>&1 | Q
echo "== blocks"; FPB_HEX_BOX_RHS=0 timeout 900 python tools/kbench.py $K 2>&1 | Q

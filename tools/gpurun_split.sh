for t in gradient_split=0 gradient_split=1; do
  echo "== $t"
  timeout 300 python tools/kbench.py --scatters auto --tune $t 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: v['ms'] for k, v in d.items() if isinstance(v, dict)})"
done

timeout 600 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "solver or pcg or spmv" 2>&1 | tail -3
timeout 300 python tools/solver_bench.py 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: {kk: round(vv, 4) if isinstance(vv, float) else vv for kk, vv in v.items()} for k, v in d.items()})"

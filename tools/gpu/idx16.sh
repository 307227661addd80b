timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/flow_probe.py 2>&1 | tail -1
timeout 600 python tools/solver_bench.py 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: (round(v['ms'],4), round(v.get('frac_hbm', 0),3), v.get('ms_per_iter')) for k,v in d.items()})"
timeout 600 python tools/c5_solver.py 2>&1 | tail -1

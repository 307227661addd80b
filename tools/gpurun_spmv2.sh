q() { python -c "import json,sys; d=json.load(sys.stdin); print({k: round(v.get('frac_hbm', v.get('ms_per_iter', 0)),4) for k, v in d.items()})"; }
echo "== staged"; timeout 300 python tools/solver_bench.py 2>&1 | q; timeout 300 python tools/c5_solver.py | tail -1
echo "== lanes-per-row"; FPB_LIB_PATH=build_variants/oldspmv/libfempack_b200.so timeout 300 python tools/solver_bench.py 2>&1 | q; FPB_LIB_PATH=build_variants/oldspmv/libfempack_b200.so timeout 300 python tools/c5_solver.py | tail -1
timeout 300 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "spmv or pcg or bicg or flow" 2>&1 | tail -1

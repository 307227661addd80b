mkdir -p gpurun_out
q() { python -c "import json,sys; d=json.load(sys.stdin); print({k: round(v.get('frac_hbm', v.get('ms_per_iter', 0)),4) for k, v in d.items()})"; }
echo "== default (R=4)"; timeout 300 python tools/solver_bench.py 2>&1 | q
for v in build_variants/spmv*/; do echo "== $v"; FPB_LIB_PATH=$v/libfempack_b200.so timeout 300 python tools/solver_bench.py 2>&1 | q; done
timeout 300 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "spmv or pcg or bicg" 2>&1 | tail -1

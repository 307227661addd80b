for v in "" build_variants/b16/libfempack_b200.so; do echo "== $v"
FPB_LIB_PATH=$v timeout 600 python tools/flow_probe.py 2>&1 | tail -1
FPB_LIB_PATH=$v timeout 600 python tools/solver_bench.py 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: (round(v['ms'],4), round(v.get('frac_hbm', 0),3), v.get('ms_per_iter')) for k,v in d.items() if k in ('spmv','pcg','bicgstab')})"
done

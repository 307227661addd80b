timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/solver_bench.py 2>&1 | tail -60
timeout 600 python tools/c5_solver.py 2>&1 | tail -20
timeout 900 python tools/spmv_probe.py 2>&1 | tail -3

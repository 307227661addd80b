timeout 300 python tools/solver_bench.py
timeout 600 python tools/solver_bench.py --nx 256 --ny 256 --nz 256

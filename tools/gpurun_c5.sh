echo "== default"; timeout 300 python tools/c5_solver.py 2>&1 | tail -1
for v in build_variants/*/; do echo "== $v"; FPB_LIB_PATH=$v/libfempack_b200.so timeout 300 python tools/c5_solver.py 2>&1 | tail -1; done

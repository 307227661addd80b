timeout 900 python tools/spmv_probe.py 2>&1 | tail -3
for v in build_variants/*/; do echo "== $v"; FPB_LIB_PATH=$v/libfempack_b200.so timeout 600 python tools/spmv_probe.py 2>&1 | tail -3; done

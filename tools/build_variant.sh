#!/bin/bash
# tools/build_variant.sh NAME "-DFOO=1 ..." : builds build_variants/NAME/libfempack_b200.so
# (development aid for A/B timing on the GPU box via FPB_LIB_PATH)
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build_variants/$name
mkdir -p $out
cd $root/paper_2107_11541_b200/csrc
for f in $(sed -n "s/^SRCS := //p" Makefile | sed "s/\.cu//g"); do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -rdc=true "$@" -c $f.cu -o $out/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $out/*.o -o $out/libfempack_b200.so -lcudart_static -ldl
echo built $out

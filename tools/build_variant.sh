#!/bin/bash
# Build a variant of liboctgpu.so with extra nvcc defines into tools/variants/NAME/
# (A/B experiments; load it with OCTGPU_LIB=tools/variants/NAME/liboctgpu.so).
#   tools/build_variant.sh NAME -DFOO=1 ...
set -e
NAME=$1; shift
HERE=$(cd "$(dirname "$0")/.." && pwd)
C=$HERE/paper_1606_00310_b200/csrc
OUT=$HERE/tools/variants/$NAME
mkdir -p $OUT
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-ffp-contract=off -I$HERE/include -I$C $*"
for f in engine kernels mcs_bulk mcs_deep measure p2p; do nvcc $FLAGS -c $C/$f.cu -o $OUT/$f.o & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/liboctgpu.so $OUT/*.o
rm -f $OUT/*.o
echo built $OUT/liboctgpu.so

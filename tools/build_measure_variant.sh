#!/bin/bash
# A/B variant of liboctgpu.so with only measure.cu rebuilt (extra nvcc defines) into tools/variants/NAME/;
# the other objects are the current in-tree build. Load with OCTGPU_LIB=tools/variants/NAME/liboctgpu.so.
set -e
NAME=$1; shift
HERE=$(cd "$(dirname "$0")/.." && pwd)
C=$HERE/paper_1606_00310_b200/csrc
OUT=$HERE/tools/variants/$NAME
mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-ffp-contract=off \
     -Xptxas -v -I$HERE/include -I$C "$@" -c $C/measure.cu -o $OUT/measure.o 2> $OUT/ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/liboctgpu.so $C/engine.o $C/kernels.o $C/mcs_bulk.o \
     $C/mcs_deep.o $OUT/measure.o $C/p2p.o
grep -A2 "k_measure_rowsImE" $OUT/ptxas.log | grep -E "registers|spill" | head -2
echo built $OUT/liboctgpu.so

#!/bin/bash
# Build liboctgpu.so of a git revision into tools/variants/git_<name>/ (A/B against the working tree).
#   tools/build_git_variant.sh REV NAME
set -e
REV=$1; NAME=$2
HERE=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/octgpu_wt_$NAME
OUT=$HERE/tools/variants/git_$NAME
rm -rf "$WT"
git -C "$HERE" worktree add -f "$WT" "$REV" > /dev/null 2>&1
mkdir -p "$OUT"
C=$WT/paper_1606_00310_b200/csrc
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-ffp-contract=off -I$WT/include -I$C"
for f in engine kernels mcs_bulk mcs_deep measure p2p; do nvcc $FLAGS -c "$C/$f.cu" -o "$OUT/$f.o" 2> /dev/null & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/liboctgpu.so" "$OUT"/engine.o "$OUT"/kernels.o \
     "$OUT"/mcs_bulk.o "$OUT"/mcs_deep.o "$OUT"/measure.o "$OUT"/p2p.o
for f in engine kernels mcs_bulk mcs_deep measure p2p; do rm -f "$OUT/$f.o"; done
git -C "$HERE" worktree remove --force "$WT"
echo built "$OUT/liboctgpu.so"

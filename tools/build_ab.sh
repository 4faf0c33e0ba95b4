#!/bin/bash
# Build an alternative libotk .so from another source tree (same ABI) for A/B timing:
#   tools/build_ab.sh <tree-with-paper_2201_12324_b200/csrc-and-include> <out.so>
set -e
SRC=$1; OUT=$2; TMP=$(mktemp -d)
for f in $SRC/paper_2201_12324_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       --expt-relaxed-constexpr -I $SRC/include -I $SRC/paper_2201_12324_b200/csrc -c $f -o $TMP/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $TMP/*.o
rm -rf $TMP

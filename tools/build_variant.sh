#!/bin/bash
# Build the library with extra nvcc flags (e.g. -DOTK_SMALL_RPG=4) for same-box A/B:
#   tools/build_variant.sh <out.so> [nvcc flags...]; then OTK_LIB=<out.so> python ...
set -e
OUT=$1; shift
ROOT=$(cd $(dirname $0)/.. && pwd); TMP=$(mktemp -d)
for f in $ROOT/paper_2201_12324_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       --expt-relaxed-constexpr "$@" -I $ROOT/include -I $ROOT/paper_2201_12324_b200/csrc \
       -c $f -o $TMP/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $TMP/*.o
rm -rf $TMP

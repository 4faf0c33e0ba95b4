#!/bin/bash
# Same-box A/B of the persistent small solve: rebuild only solve_small.cu with
# extra nvcc flags and link it with the library's other objects.
#   tools/variant_small.sh <out.so> [-DOTK_ER_PAIRS=8 ...]; then OTK_LIB=<out.so> python ...
set -e
OUT=$1; shift
ROOT=$(cd $(dirname $0)/.. && pwd); P=$ROOT/paper_2201_12324_b200; TMP=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
     --expt-relaxed-constexpr --split-compile 0 "$@" -I $ROOT/include -I $P/csrc \
     -c $P/csrc/solve_small.cu -o $TMP/solve_small.o
OBJS=$(ls $P/build_obj/*.o | grep -v solve_small.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $OBJS $TMP/solve_small.o
rm -rf $TMP

#!/bin/bash
# Experimental engine variant: recompile kernels.cu (or SRC=<name> of another
# csrc/*.cu) with extra nvcc flags and
# link it with the regular objects into exp_libs/libtsv_<name>.so; select it
# at run time with TSV_LIB=exp_libs/libtsv_<name>.so.
# Usage: tools/build_variant.sh <name> <nvcc flags...>
#   e.g. tools/build_variant.sh m4 '-DTSV_WIDE_MINB(P)=4'
set -e
cd "$(dirname "$0")/.."
name=$1; shift
P=paper_2001_07158_b200
make -s -C $P >/dev/null
mkdir -p exp_libs build_exp
src=${SRC:-kernels}
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xptxas -v \
  -Xcompiler -fPIC,-fopenmp -ccbin g++ "$@" -c $P/csrc/$src.cu -o build_exp/${src}_$name.o \
  2> build_exp/${src}_$name.ptxas.log
objs=""
for o in $P/build/*.o; do
  [ "$(basename $o .o)" = "$src" ] && objs="$objs build_exp/${src}_$name.o" || objs="$objs $o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp_libs/libtsv_$name.so \
  $objs -Xcompiler -fopenmp -lgomp
grep -A2 "k_level_wideILi2ELb0ELb1ELb0" build_exp/${src}_$name.ptxas.log | grep -E "registers|spill" | head -2

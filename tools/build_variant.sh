#!/bin/bash
# Experimental engine variant: recompile kernels.cu with extra nvcc flags and
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
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xptxas -v \
  -Xcompiler -fPIC,-fopenmp -ccbin g++ "$@" -c $P/csrc/kernels.cu -o build_exp/kernels_$name.o \
  2> build_exp/kernels_$name.ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp_libs/libtsv_$name.so \
  build_exp/kernels_$name.o $P/build/static_kernels.o $P/build/build_kernels.o \
  $P/build/gf_bench.o $P/build/tsv_abi.o $P/build/layout.o -Xcompiler -fopenmp -lgomp
grep -A2 "k_level_wideILi2ELb0ELb1ELb0" build_exp/kernels_$name.ptxas.log | grep -E "registers|spill" | head -2

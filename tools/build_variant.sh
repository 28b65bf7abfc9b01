#!/bin/bash
# Build a variant of libblockeig_b200.so with spmm.cu compiled under extra -D flags:
#   tools/build_variant.sh <name> -DBE_SPMM_MINB=3 ...   -> tools/bin/lib_<name>.so
set -e
name=$1; shift
SRC=${SRC:-spmm}   # which csrc/<SRC>.cu gets the extra flags
ROOT=$(cd "$(dirname "$0")/.." && pwd)
O=$ROOT/build/obj
mkdir -p $ROOT/tools/bin
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -Xcompiler -fPIC,-pthread -I $ROOT/include -I $ROOT/paper_2109_00485_b200/csrc \
  -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr "$@" \
  -c $ROOT/paper_2109_00485_b200/csrc/$SRC.cu -o /tmp/${SRC}_$name.o
objs=$(ls $O/*.o | grep -v $SRC.cu.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/tools/bin/lib_$name.so /tmp/${SRC}_$name.o $objs \
  -L/usr/local/cuda/lib64 -lcudart -lcusolver -lcublas -ldl -lpthread
echo built tools/bin/lib_$name.so

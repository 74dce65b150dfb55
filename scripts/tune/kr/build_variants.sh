#!/bin/bash
# KR tiles-per-CTA sweep (tuning only): relink libswdft2d.so with kr_rows.cu compiled for
# several KR_PER32 / KR_PER64 values into scripts/tune/kr/_build/libswdft2d_<p32>_<p64>.so
set -e
cd "$(dirname "$0")/../../.."
B=paper_1707_08213_b200/_build
mkdir -p scripts/tune/kr/_build
for v in "8192 4096" "16384 8192" "32768 16384" "65536 8192"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -DKR_PER32=$1 -DKR_PER64=$2 -c paper_1707_08213_b200/csrc/kr_rows.cu -o scripts/tune/kr/_build/kr_$1.o
  objs=$(ls $B/*.o | grep -v kr_rows.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
    -Xlinker --version-script=paper_1707_08213_b200/csrc/exports.map \
    -o scripts/tune/kr/_build/libswdft2d_$1_$2.so $objs scripts/tune/kr/_build/kr_$1.o
done
ls scripts/tune/kr/_build/*.so

#!/bin/bash
# K1 store-policy experiment (tuning only): libswdft2d.so relinked with the K1 units
# compiled with -DK1_PLAIN_STORES -> scripts/tune/k1store/_build/libswdft2d_plain.so
set -e
cd "$(dirname "$0")/../../.."
B=paper_1707_08213_b200/_build
O=scripts/tune/k1store/_build
for m0 in 0 1 2 3 4 5 6 7 8 9; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -DK1_PLAIN_STORES -DK1_M0=$m0 -c paper_1707_08213_b200/csrc/k1_inst.cu -o $O/k1_m0_$m0.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -Xlinker --version-script=paper_1707_08213_b200/csrc/exports.map -o $O/libswdft2d_plain.so \
  $B/abi.o $B/k0_window.o $B/k2_push.o $B/kr_rows.o $O/k1_m0_*.o

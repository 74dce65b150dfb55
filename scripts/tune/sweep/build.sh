#!/bin/bash
# builds scripts/tune/sweep/_build/libsweep.so (tuning harness; not product code)
set -e
cd "$(dirname "$0")"
mkdir -p _build
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I ../../../include -I ../../../paper_1707_08213_b200/csrc"
for f in sweep_main.cu sweep64.cu sweep_m0_2.cu sweep_m0_3.cu sweep_m0_4.cu sweep_m0_5.cu sweep_m0_6.cu sweep_m0_7.cu; do
  nvcc $F -c $f -o _build/${f%.cu}.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o _build/libsweep.so _build/*.o

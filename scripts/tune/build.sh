#!/bin/bash
# builds scripts/tune/_build/libtune.so (tuning harness; not product code)
set -e
cd "$(dirname "$0")"
mkdir -p _build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I ../../include -I ../../paper_1707_08213_b200/csrc -DSWDFT2D_K1_MAX_M0=10 -shared -cudart static \
  -Xptxas -v -o _build/libtune.so tune_k1.cu 2> _build/ptxas.log
grep -A1 "Function properties for _ZN7swdft2d16k1" _build/ptxas.log | grep -E "spill|registers" | head -40 || true
grep -E "Used [0-9]+ registers" _build/ptxas.log | head -40

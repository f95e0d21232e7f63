#!/bin/bash
# build the current working tree's library as tools/exp/lib_B.so (for ab_bench.sh)
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/exp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -Xcompiler -fPIC \
  -shared -o tools/exp/lib_B.so paper_1806_04960_b200/csrc/wb_capi.cu 2>/dev/null

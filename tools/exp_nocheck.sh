#!/bin/bash
# Measurement experiment: the cost of the exactness checks of the speculative
# divisions.  Builds the library with the range checks compiled out (results
# are no longer guaranteed bit-exact for out-of-range operands; never
# shipped) into tools/exp/.  Time it with
#   WB_LIB_PATH=tools/exp/lib_NOCHECK.so VARIANTS=6 python tools/variant_bench.py
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/exp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -Xcompiler -fPIC \
  -shared -DWB_EXPERIMENT_NOCHECK -o tools/exp/lib_NOCHECK.so \
  paper_1806_04960_b200/csrc/wb_capi.cu 2>/dev/null
ls tools/exp

#!/bin/bash
# Measurement experiment: the cost of the exactness checks of the speculative
# divisions.  Builds the library with the checks compiled out (results are no
# longer guaranteed bit-exact for out-of-range operands; never shipped) into
# tools/exp/: all checks, only the general-division checks, only the
# constant-divisor checks.  Time with WB_LIB_PATH=tools/exp/<lib> tools/variant_bench.py.
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/exp
for v in NOCHECK NOCHECK_DIV NOCHECK_DIVC; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -Xcompiler -fPIC \
    -shared -DWB_EXPERIMENT_$v -o tools/exp/lib_$v.so paper_1806_04960_b200/csrc/wb_capi.cu \
    2>/dev/null &
done
wait
ls tools/exp

#!/bin/bash
# build the working tree's library with extra nvcc flags into tools/exp/lib_<name>.so
# usage: tools/build_variant.sh <name> [nvcc flags...]   (A/B experiments, tools/ab_libs.py)
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/exp
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -lineinfo -std=c++17 -Xcompiler -fPIC \
  -shared "$@" -o tools/exp/lib_$name.so paper_1806_04960_b200/csrc/wb_capi.cu -Xptxas -v 2>&1 | \
  grep -A2 "k_stepILi128ELi3ELb1ELb0" | grep -E "Used|spill" | tr '\n' ' '; echo " -> lib_$name.so"

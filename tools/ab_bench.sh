#!/bin/bash
# A/B timing of k_step on one box: the in-tree library (A) against
# tools/exp/lib_B.so (B, built from a modified tree by tools/build_b.sh),
# alternating.  WB_VB_WARM=N times the kernel after N steps (default 3).
# usage (on the GPU box): bash tools/ab_bench.sh [rounds]
n=${1:-3}
for i in $(seq $n); do
  echo -n "A "; VARIANTS=6 python tools/variant_bench.py 2>&1 | tail -1
  echo -n "B "; WB_LIB_PATH=tools/exp/lib_B.so VARIANTS=6 python tools/variant_bench.py 2>&1 | tail -1
done

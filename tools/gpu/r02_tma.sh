# TMA-staged k_step: A/B timing against the round-1 kernel, then the GPU suite
set -x
for w in 3 300; do
  WB_VB_WARM=$w VARIANTS=3,6,0 timeout 600 python tools/variant_bench.py 2>&1 | tail -3
  WB_VB_WARM=$w WB_LIB_PATH=tools/exp/lib_r01.so VARIANTS=6 timeout 600 python tools/variant_bench.py 2>&1 | tail -1
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_tma_gputest.log 2>&1; tail -15 gpurun_out/r02_tma_gputest.log

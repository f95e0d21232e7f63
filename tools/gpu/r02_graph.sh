timeout 300 python -m pytest tests/test_gpu_distributed.py -q -x -k "nccl_world1" 2>&1 | grep -E "Error|error|assert|passed|failed|Warning" | head -30
LIBS="lim=tools/exp/lib_lim.so,ysm=tools/exp/lib_ysm.so" timeout 900 python tools/ab_libs.py 2 3,300 | tail -8

timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_slabs.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3
timeout 600 python tools/overlap_bench.py 20

timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02_full_gputest.log 2>&1; tail -3 gpurun_out/r02_full_gputest.log
python bench.py > gpurun_out/r02_b2.json 2> gpurun_out/r02_b2.err; tail -2 gpurun_out/r02_b2.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err; tail -2 gpurun_out/r02_ref.err
python __graft_entry__.py 2>&1 | tail -1

# round-2 validation of the current tree: GPU tests, bench line, reference arm, smoke, launch list
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02_full2_gputest.log 2>&1; tail -3 gpurun_out/r02_full2_gputest.log
python bench.py > gpurun_out/r02_b3.json 2> gpurun_out/r02_b3.err; tail -2 gpurun_out/r02_b3.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_ref3.json 2> gpurun_out/r02_ref3.err; tail -2 gpurun_out/r02_ref3.err
python __graft_entry__.py 2>&1 | tail -1
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-developed"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches3.csv $CMD > gpurun_out/r02_ncu31.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/r02_kstep3 $CMD > gpurun_out/r02_ncu32.log 2>&1
echo "ncu rc=$?"

# launch list + one full capture of k_step (bench workload, step 4)
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-developed"
$CMD > gpurun_out/r02_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/r02_kstep $CMD > gpurun_out/r02_ncu2.log 2>&1
echo "rc=$?"
tail -2 gpurun_out/r02_ncu2.log

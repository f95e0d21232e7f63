# one full ncu capture of k_step in the developed flow (step 301 of the bench slab)
timeout 300 python tools/dev_step.py 300 > gpurun_out/r02_dev300.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_step -s 301 -c 1 -o gpurun_out/r02_kstep300 python tools/dev_step.py 300 > gpurun_out/r02_ncu300.log 2>&1
echo "rc=$?"; cat gpurun_out/r02_dev300.log; tail -3 gpurun_out/r02_ncu300.log

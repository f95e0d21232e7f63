# final round-2 bench line (N=1) and the N>1 bench path exercised with two ranks on one GPU (gloo)
python bench.py > gpurun_out/r02_b4.json 2> gpurun_out/r02_b4.err; tail -2 gpurun_out/r02_b4.err
WB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 > gpurun_out/r02_b4_n2.json 2> gpurun_out/r02_b4_n2.err; echo "n2 rc=$?"; tail -3 gpurun_out/r02_b4_n2.err

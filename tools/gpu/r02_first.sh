set -x
nproc; free -g; lscpu | head -20; nvidia-smi --query-gpu=name,memory.total --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py > gpurun_out/r02_b0.json 2> gpurun_out/r02_b0.err; tail -3 gpurun_out/r02_b0.err
cat gpurun_out/r02_b0.json

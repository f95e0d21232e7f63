# round 2: parity suite (incl. full-size oracle lockstep, forced replay), bench, sanitizers
set -x
python -m pytest tests -m gpu -q -x -rs --durations=15 > gpurun_out/r02_gputest.log 2>&1; tail -30 gpurun_out/r02_gputest.log
python bench.py > gpurun_out/r02_b1.json 2> gpurun_out/r02_b1.err; tail -3 gpurun_out/r02_b1.err; cat gpurun_out/r02_b1.json
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_case.py > gpurun_out/r02_sanitize_$t.log 2>&1; echo "$t rc=$?"; tail -4 gpurun_out/r02_sanitize_$t.log
done

export CUDA_LAUNCH_BLOCKING=1
for v in 0 3 5 6 7; do for res in "96,48" "130,70" "1024,512"; do
WB_KSTEP_VARIANT=$v timeout 300 python -c "
from paper_1806_04960_b200.scenarios import build_scenario
from paper_1806_04960_b200.timestepper import Simulation
sc = build_scenario('wall-impact', ($res))
sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
try:
    sim.advance(); sim.run_steps(2); print('variant $v res $res OK', sim.step_count)
except Exception as e:
    print('variant $v res $res FAIL', e)
" 2>&1 | tail -1
done; done

"""Small device run for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("WB_FUSE_DETECT", "1")
from paper_1806_04960_b200.scenarios import build_scenario  # noqa: E402
from paper_1806_04960_b200.timestepper import Simulation  # noqa: E402

for name, res in (("wall-impact", (130, 70)), ("jet", (96, 64)), ("dambreak-step-wet", (120, 40))):
    sc = build_scenario(name, res)
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary, rows_per_block=16)
    for _ in range(3):
        sim.advance()
    sim.run_steps(4, chunk=2)
    d = Simulation(sc.grid, sc.params, sc.q0, sc.boundary, debug=True)
    d.advance()
    print(name, sim.step_count, sim.t, d.step_count, flush=True)
print("sanitize case OK")

"""Where the exact replays happen in a developed flow (GPU): advances the C5
slab N steps and prints the per-kind replay counts of the next 5 steps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1806_04960_b200.scenarios import build_scenario  # noqa: E402
from paper_1806_04960_b200.timestepper import Simulation  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
sc = build_scenario("wall-impact", (4096, 16384))
sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
for target in (3, 100, 200, n):
    sim.run_steps(target - sim.step_count, chunk=16)
    a = sim.work_counters()["replays_by_kind"]
    sim.run_steps(5, chunk=5)
    b = sim.work_counters()
    d = {k: (b["replays_by_kind"][k] - a[k]) / 5 for k in a}
    print(f"step {target}: replays per step " + ", ".join(f"{k} {v:.3g}" for k, v in d.items()),
          f"| x_faces {b['x_faces']:.3g} n2nd {b['n_second_order']:.3g}", flush=True)

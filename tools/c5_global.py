"""The full C5 global grid (32768 x 16384 = 5.4e8 cells, 2 x 17 GB of state
planes) on ONE B200: build, upload, 5 steps, mass check, device memory used."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1806_04960_b200.scenarios import build_scenario  # noqa: E402
from paper_1806_04960_b200.timestepper import Simulation  # noqa: E402

t0 = time.perf_counter()
sc = build_scenario("wall-impact", (32768, 16384))
t1 = time.perf_counter()
sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
del sc
t2 = time.perf_counter()
free, total = torch.cuda.mem_get_info()
m0 = sim.total_mass(device=True)
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
sim.run_steps(2)
torch.cuda.synchronize()
s.record()
sim.run_steps(5)
e.record()
torch.cuda.synchronize()
m1 = sim.total_mass(device=True)
print(f"build {t1 - t0:.1f} s, upload {t2 - t1:.1f} s, device memory in use "
      f"{(total - free) / 1e9:.1f} of {total / 1e9:.1f} GB, {s.elapsed_time(e) / 5:.2f} ms/step "
      f"({5.37e8 * 5 / (s.elapsed_time(e) * 1e-3):.3g} cell-updates/s), "
      f"mass drift {abs(m1 - m0) / m0:.2e}", flush=True)

"""Host<->device transfer rates of the e2e leg (GPU): raw pinned cudaMemcpy
(torch) against wb_set_state / wb_get_state of the bench slab."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_04960_b200.scenarios import build_scenario  # noqa: E402
from paper_1806_04960_b200.timestepper import Simulation  # noqa: E402

nx, ny = 4096, 16384
nbytes = nx * ny * 5 * 8
h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
d = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
for name, f in (("raw H2D", lambda: d.copy_(h, non_blocking=True)),
                ("raw D2H", lambda: h.copy_(d, non_blocking=True))):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"{name}: {nbytes / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms for {nbytes / 1e9:.2f} GB)")
del d
sc = build_scenario("wall-impact", (nx, ny))
q_host = torch.empty((nx, ny, 5), dtype=torch.float64, pin_memory=True).numpy()
q_host[...] = sc.q0
out = torch.empty((nx, ny, 5), dtype=torch.float64, pin_memory=True).numpy()
sim = Simulation(sc.grid, sc.params, q_host, sc.boundary)
for name, f in (("wb_set_state", lambda: setattr(sim, "q", q_host)),
                ("wb_get_state", lambda: sim.get_state(out=out))):
    f()
    t0 = time.perf_counter()
    for _ in range(3):
        f()
    dt = (time.perf_counter() - t0) / 3
    print(f"{name}: {nbytes / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms)")
t0 = time.perf_counter()
for _ in range(20):
    sim.advance()
print(f"20 x advance(): {(time.perf_counter() - t0) * 1e3:.1f} ms")

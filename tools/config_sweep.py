"""Throughput of the device path on the BASELINE.json configurations (GPU).
python tools/config_sweep.py [steps]"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1806_04960_b200 import _lib  # noqa: E402
from paper_1806_04960_b200.scenarios import build_scenario  # noqa: E402
from paper_1806_04960_b200.timestepper import Simulation  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
only = sys.argv[3].split(",") if len(sys.argv) > 3 else None
CONFIGS = [("C1 dambreak-dry", "dambreak-dry", (200, 100)),
           ("C2 lake", "lake", (2048, 1024)),
           ("C3 drop", "drop", (4096, 4096)),
           ("C4 weir", "weir", (16384, 8192)),
           ("C5 wall-impact slab", "wall-impact", (4096, 16384))]
for label, name, res in CONFIGS:
    if only and label.split()[0] not in only:
        continue
    t0 = time.perf_counter()
    sc = build_scenario(name, res)
    tb = time.perf_counter() - t0
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
    s = torch.cuda.Stream()
    _lib.check(sim._L.wb_set_stream(sim._h, ctypes.c_void_p(s.cuda_stream)), "stream")
    sim.run_steps(warm, chunk=max(d for d in range(1, 17) if warm % d == 0))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    sim.run_steps(steps, chunk=max(d for d in range(1, 17) if steps % d == 0))
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    n = sc.grid.fluid_cell_count()
    wc = sim.work_counters()
    print(f"{label:22s} {res[0]}x{res[1]} after {warm} steps: {ms:8.3f} ms/step  {n / ms / 1e6:9.3f} Gcell/s  "
          f"(2nd={wc['n_second_order']}, Ex={wc['x_faces']}, Ey={wc['y_faces']}; IC {tb:.1f}s)",
          flush=True)
    del sim

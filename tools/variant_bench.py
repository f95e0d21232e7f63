"""Time k_step launch variants (occupancy experiments) on the bench workload
and check they are bit-identical.  GPU.  python tools/variant_bench.py [nx ny]"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1806_04960_b200 import _lib  # noqa: E402
from paper_1806_04960_b200.scenarios import build_scenario  # noqa: E402
from paper_1806_04960_b200.timestepper import Simulation  # noqa: E402

nx, ny = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4096, 16384)
variants = [int(v) for v in os.environ.get("VARIANTS", "0,1,2,3,4,5").split(",")]
sc = build_scenario("wall-impact", (nx, ny))
ref = None
for v in variants:
    os.environ["WB_KSTEP_VARIANT"] = str(v)
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
    warm = int(os.environ.get("WB_VB_WARM", "3"))
    sim.run_steps(warm, chunk=min(warm, 16))
    md, ms, mt = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _lib.check(sim._L.wb_profile_steps(sim._h, 5, ctypes.byref(md), ctypes.byref(ms),
                                       ctypes.byref(mt)), "profile")
    q = sim.q
    same = "ref" if ref is None else ("same" if np.array_equal(q, ref) else "DIFFERENT")
    if ref is None:
        ref = q
    print(f"variant {v}: k_step {ms.value:.3f} ms  detect {md.value:.3f} ms  "
          f"pipeline {mt.value:.3f} ms  [{same}]", flush=True)
    del sim

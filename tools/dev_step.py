"""Advance the bench slab (wall-impact C5, 4096x16384) `warm` steps, then time
k_step alone over 3 steps (wb_profile_steps).  Used to capture one k_step of
the developed flow under ncu:

    ncu --set full -k regex:k_step -s 301 -c 1 python tools/dev_step.py 300
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_04960_b200 import _lib  # noqa: E402
from paper_1806_04960_b200.scenarios import build_scenario  # noqa: E402
from paper_1806_04960_b200.timestepper import Simulation  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 300
sc = build_scenario("wall-impact", (4096, 16384), host_state=False)
sim = Simulation.from_scenario(sc, device=0)
sim.run_steps(warm, chunk=max(d for d in range(1, 17) if warm % d == 0))
md, ms, mt = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
_lib.check(sim._L.wb_profile_steps(sim._h, 3, ctypes.byref(md), ctypes.byref(ms),
                                   ctypes.byref(mt)), "profile")
print(f"warm {warm}: k_step {ms.value:.3f} ms  counters {sim.work_counters()}")

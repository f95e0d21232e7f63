"""Step-by-step stage comparison of the device path against the oracle
(debug aid; GPU).  Usage: python tools/debug_parity.py scenario nx ny steps"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as orc  # noqa: E402
from paper_1806_04960_b200.scenarios import build_scenario  # noqa: E402
from paper_1806_04960_b200.timestepper import Simulation  # noqa: E402

STAGES = ("rhoE_c", "rhoE_fy", "quiet", "psi", "fW", "fE", "fS", "fN", "vol", "DW", "DE",
          "DS", "DN")


def main():
    name, nx, ny, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    sc = build_scenario(name, (nx, ny))
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary, debug=True)
    ref = orc.OracleSimulation(sc.grid, sc.params, sc.q0, sc.boundary)
    fl = sc.grid.mask != 0
    for s in range(1, steps + 1):
        qprev = ref.q.copy()
        dtr = ref.advance()
        dtg = sim.advance()
        print(f"step {s}: dt {'==' if dtr == dtg else '!='} ({dtr!r} {dtg!r})")
        if not (np.array_equal(sim.y0s, ref.y0s) and np.array_equal(sim.aeqs, ref.aeqs)):
            d = np.nonzero((sim.y0s != ref.y0s) | (sim.aeqs != ref.aeqs))[0]
            print("  columns differ:", d[:10], sim.y0s[d[:3]], ref.y0s[d[:3]])
        bad = False
        for k in STAGES:
            g, r = getattr(sim, k), getattr(ref, k)
            if k in ("rhoE_fy",):
                diff = g != r
            else:
                diff = (g != r) & (fl[..., None] if g.ndim == 3 else fl)
            if diff.any():
                idx = np.argwhere(diff)
                i0 = tuple(idx[0])
                print(f"  stage {k}: {len(idx)} diffs; first {i0}: gpu {g[i0]!r} ref {r[i0]!r}")
                c = i0[:2]
                print("    quiet g/r", sim.quiet[c], ref.quiet[c], " psi g", sim.psi[c], "r", ref.psi[c])
                print("    q_prev", qprev[c])
                bad = True
        q = sim.q
        if not np.array_equal(q, ref.q):
            idx = np.argwhere(q != ref.q)
            print(f"  q: {len(idx)} diffs; first {tuple(idx[0])}: {q[tuple(idx[0])]!r} "
                  f"{ref.q[tuple(idx[0])]!r}")
            bad = True
        if bad:
            break


if __name__ == "__main__":
    main()

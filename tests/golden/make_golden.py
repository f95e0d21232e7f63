"""Generate the golden fixtures that pin the CPU oracle to the real reference.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the UNMODIFIED reference package ``wbflow`` from /root/reference
and runs its own scalar kernels and its own ``Simulation`` (Numba CPU path) on
deterministic inputs built by ``paper_1806_04960_b200.scenarios``.  Outputs go
to tests/golden/*.npz (committed).  Nothing at test time reads /root/reference.
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from wbflow import kernels as K  # noqa: E402  (the reference)
from wbflow import timestepper as TS  # noqa: E402
from wbflow.errors import SimulationError as RefSimError  # noqa: E402
from wbflow.grid import BoundaryCondition as RefBC, BoundarySpec as RefBS  # noqa: E402

from paper_1806_04960_b200.scenarios import build_scenario  # noqa: E402

STAGES = ("y0s", "aeqs", "rhoE_c", "rhoE_fy", "fW", "fE", "fS", "fN", "vol", "psi",
          "quiet", "DW", "DE", "DS", "DN")


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_boundary(b):
    conv = lambda c: RefBC(c.kind, c.state, c.segment)  # noqa: E731
    return RefBS(conv(b.left), conv(b.right), conv(b.bottom), conv(b.top))


def ref_sim(sc):
    return TS.Simulation(sc.grid, sc.params, sc.q0, ref_boundary(sc.boundary), cfl=0.45,
                         workers=8)


def random_states(rng, n, k0, rho0, eps):
    c = np.sqrt(k0 / rho0)
    a = rng.uniform(eps, 1 - eps, n)
    rho = rng.uniform(0.9, 1.1, n) * rho0
    u = rng.uniform(-0.5, 0.5, n) * c
    v = rng.uniform(-0.5, 0.5, n) * c
    y = rng.uniform(0.0, 2.0, n)
    return np.stack([a * rho, a * rho * u, a * rho * v, a, y], axis=1)


def scalar_fixtures():
    rng = np.random.default_rng(12345)
    out = {}
    k0, rho0, g = 2.78e5, 1000.0, 9.81
    n = 2000
    qm = random_states(rng, n, k0, rho0, 1e-3)
    qp = random_states(rng, n, k0, rho0, 1e-3)
    qp[: n // 2, 4] = qm[: n // 2, 4]           # half with equal heights
    qp[-5:] = qm[-5:]                           # identical pairs -> exact zeros
    # second-half states: small fluctuations about a common state (near-quiet edges)
    qp[n // 2:n // 2 + 200, :4] = qm[n // 2:n // 2 + 200, :4] * (1 + 1e-9 * rng.standard_normal((200, 4)))
    out["x_qm"], out["x_qp"] = qm, qp
    out["x_out"] = np.array([K.osher_x_edge(*qm[e], *qp[e], k0, rho0, 1.0) for e in range(n)])
    out["x_out_g7"] = np.array([K.osher_x_edge(*qm[e], *qp[e], k0, rho0, 7.0)
                                for e in range(200)])
    y0 = rng.uniform(0.5, 2.5, n)
    aeq = rng.choice([1.0, 1 - 1e-3, 1e-3], n)
    out["y_y0"], out["y_aeq"] = y0, aeq
    out["y_out"] = np.array([K.or_y_edge(*qm[e], *qp[e], y0[e], aeq[e], k0, rho0, 1.0, g)
                             for e in range(n)])
    out["y_out_g7"] = np.array([K.or_y_edge(*qm[e], *qp[e], y0[e], aeq[e], k0, rho0, 7.0, g)
                                for e in range(200)])
    ys = rng.uniform(-3.0, 3.0, 20000)
    y0s = rng.uniform(-3.0, 3.0, 20000)
    ks = rng.choice([2.25e9, 6.37e5, 2.78e5, 2.62e5], 20000)
    out["e_y"], out["e_y0"], out["e_k0"] = ys, y0s, ks
    out["e_out"] = np.array([K.eq_rho(ys[e], y0s[e], ks[e], rho0, g) for e in range(20000)])
    rhos = rng.uniform(500.0, 2000.0, 500)
    out["t_rho"] = rhos
    out["t_out_g7"] = np.array([K.tait_p(r, 3e5, rho0, 7.0) for r in rhos])
    out["c_out_g7"] = np.array([K.sound_c2(r, 3e5, rho0, 7.0) for r in rhos])
    np.savez_compressed(os.path.join(HERE, "scalar_kernels.npz"), **out)


CASES = [
    # name, scenario, resolution, stage dump, full-q checkpoints, hash checkpoints, extra
    ("drop_64", "drop", (64, 64), True, (1, 50), (), {}),
    ("impact_64x36", "wall-impact", (64, 36), True, (1, 100), (), {}),
    ("plake_48", "perturbed-lake", (48, 48), True, (1, 40), (), {"seed": 3}),
    ("weir_120x40", "weir", (120, 40), False, (60,), (), {}),
    ("jet_96x64", "jet", (96, 64), True, (60,), (), {}),
    ("tait7_64x32", "tait7", (64, 32), True, (30,), (), {}),
    ("lake_64x32", "lake", (64, 32), False, (200,), (), {}),
    ("impact_200x100", "wall-impact", (200, 100), False, (), (1, 50, 150), {}),
    ("stepwet_200x40", "dambreak-step-wet", (200, 40), True, (1, 40), (), {}),
    ("spinsq_48", "spinning-square", (48, 48), True, (1, 30), (), {}),
    ("jetplate_56x40", "jet-plate", (56, 40), False, (30,), (), {}),
    ("eqflat_100", "equilibrium-flat", (100, 100), False, (100,), (), {}),
    ("dambreak_200x100", "dambreak-dry", (200, 100), False, (), (1, 10, 100, 250),
     {"run_to_error": 400}),
]


def case_fixture(name, scen, res, stages, full_at, hash_at, extra):
    sc = build_scenario(scen, res, seed=extra.get("seed", 0))
    sim = ref_sim(sc)
    out = {"q0_sha": digest(sc.q0), "dts": []}
    arrays = {}
    last = max(list(full_at) + list(hash_at) + [extra.get("run_to_error", 0)])
    err = None
    for s in range(1, last + 1):
        try:
            dt = sim.advance()
        except RefSimError as e:
            err = {"message": str(e), "step": e.step, "cell": list(e.cell) if e.cell else None}
            break
        out["dts"].append(dt)
        if s == 1 and stages:
            for k in STAGES:
                arrays["s1_" + k] = np.array(getattr(sim, k))
        if s in full_at:
            arrays[f"q_{s}"] = sim.q.copy()
        if s in hash_at:
            out[f"q_{s}_sha"] = digest(sim.q)
            arrays[f"q_{s}_summary"] = np.array([np.abs(sim.q[..., m]).sum() for m in range(5)])
    out["error"] = err
    out["steps_done"] = sim.step_count
    arrays["dts"] = np.array(out["dts"])
    meta = {k: v for k, v in out.items() if k != "dts"}
    meta.update({"scenario": scen, "resolution": list(res), "seed": extra.get("seed", 0)})
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, f"case_{name}.npz"), **arrays)
    print(name, "steps", sim.step_count, "error", err)


if __name__ == "__main__":
    only = sys.argv[1:]
    if not only:
        scalar_fixtures()
    for c in CASES:
        if not only or c[0] in only:
            case_fixture(*c)

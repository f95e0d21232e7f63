"""Pin the CPU oracle (oracle/wb_oracle.c) to the real reference.

The fixtures under tests/golden were produced by running the unmodified
reference (``wbflow`` Numba kernels and ``Simulation``) in the build
container; the oracle must reproduce them bit for bit.
"""
import numpy as np
import pytest

from golden_util import load_case, case_names, digest, same, STAGES, GOLDEN
from paper_1806_04960_b200.scenarios import build_scenario

import os


@pytest.fixture(scope="module")
def scal():
    return np.load(os.path.join(GOLDEN, "scalar_kernels.npz"))


def test_eq_rho_bitexact(oracle, scal):
    out = np.array([oracle.eq_rho(y, y0, k, 1000.0, 9.81)
                    for y, y0, k in zip(scal["e_y"], scal["e_y0"], scal["e_k0"])])
    assert same(out, scal["e_out"])


def test_tait_gamma7(oracle, scal):
    out = np.array([oracle.tait_p(r, 3e5, 1000.0, 7.0) for r in scal["t_rho"]])
    assert same(out, scal["t_out_g7"])


def test_osher_x_edge_bitexact(oracle, scal):
    qm, qp = scal["x_qm"], scal["x_qp"]
    out = np.array([oracle.osher_x_edge(qm[e], qp[e], 2.78e5, 1000.0, 1.0)
                    for e in range(len(qm))])
    assert same(out, scal["x_out"])
    assert np.all(out[-5:] == 0.0)          # D(q, q) = 0 exactly
    out7 = np.array([oracle.osher_x_edge(qm[e], qp[e], 2.78e5, 1000.0, 7.0)
                     for e in range(200)])
    assert same(out7, scal["x_out_g7"])


def test_or_y_edge_bitexact(oracle, scal):
    qm, qp = scal["x_qm"], scal["x_qp"]
    out = np.array([oracle.or_y_edge(qm[e], qp[e], scal["y_y0"][e], scal["y_aeq"][e],
                                     2.78e5, 1000.0, 1.0, 9.81) for e in range(len(qm))])
    assert same(out, scal["y_out"])
    out7 = np.array([oracle.or_y_edge(qm[e], qp[e], scal["y_y0"][e], scal["y_aeq"][e],
                                      2.78e5, 1000.0, 7.0, 9.81) for e in range(200)])
    assert same(out7, scal["y_out_g7"])


@pytest.mark.parametrize("name", case_names())
def test_oracle_trajectory(oracle, name):
    meta, arr = load_case(name)
    sc = build_scenario(meta["scenario"], tuple(meta["resolution"]), seed=meta["seed"])
    assert digest(sc.q0) == meta["q0_sha"], "scenario builder drifted from the fixture"
    sim = oracle.OracleSimulation(sc.grid, sc.params, sc.q0, sc.boundary, cfl=0.45)
    want_err = meta["error"]
    last = meta["steps_done"] + (1 if want_err else 0)
    err = None
    for s in range(1, last + 1):
        try:
            sim.advance()
        except oracle.OracleError as e:
            err = e
            break
        if s == 1 and "s1_fW" in arr:
            for k in STAGES:
                assert same(getattr(sim, k), arr["s1_" + k]), f"stage {k} differs"
        if f"q_{s}" in arr:
            assert same(sim.q, arr[f"q_{s}"]), f"q differs at step {s}"
        if f"q_{s}_sha" in meta:
            assert digest(sim.q) == meta[f"q_{s}_sha"], f"q hash differs at step {s}"
    assert same(np.array(sim.dt_log), arr["dts"])
    if want_err:
        assert err is not None, "reference aborted but oracle did not"
        assert str(err) == want_err["message"]
        assert err.step == want_err["step"] and list(err.cell) == want_err["cell"]
    else:
        assert err is None


def test_oracle_thread_invariance(oracle):
    """Bit-identical for any worker count (timestepper.py:27-30)."""
    sc = build_scenario("perturbed-lake", (40, 40), seed=1)
    res = []
    for n in (1, 4):
        oracle.set_threads(n)
        sim = oracle.OracleSimulation(sc.grid, sc.params, sc.q0, sc.boundary)
        sim.run_steps(5)
        res.append(sim.q.copy())
    oracle.set_threads(os.cpu_count())
    assert same(res[0], res[1])

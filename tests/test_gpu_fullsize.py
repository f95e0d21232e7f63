"""Size-independent properties at BASELINE.json's full sizes (GPU tests).

The CPU oracle cannot run these sizes in test time, so parity is checked
through properties that must hold bit for bit:
- x-slab decomposition equivalence at C4 size (16384 x 8192): 3 device slabs
  against the single-domain handle;
- launch-configuration invariance at C5 slab size (4096 x 16384);
- mass conservation on C3 (4096^2, reflective walls);
- C2 lake at rest stays bit-identical for 1000 steps.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("overlap", [False, True])
def test_c4_weir_slabs_equal_single(torch_cuda, overlap):
    from test_gpu_slabs import _run, _slabs
    from paper_1806_04960_b200.scenarios import build_scenario
    from paper_1806_04960_b200.timestepper import Simulation
    res = (16384, 8192)
    slabs = _slabs(torch_cuda, "weir", res, 3)
    assert _run(torch_cuda, slabs, 4, overlap=overlap) is None
    q_slabs = np.concatenate([s.owned_state() for s in slabs], axis=0)
    t_slabs = slabs[0].status()["t"]
    del slabs
    sc = build_scenario("weir", res)
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
    sim.run_steps(4)
    assert sim.t == t_slabs
    assert np.array_equal(sim.q, q_slabs)


def test_c5_launch_variants_equal(torch_cuda, monkeypatch):
    from paper_1806_04960_b200.scenarios import build_scenario
    from paper_1806_04960_b200.timestepper import Simulation
    sc = build_scenario("wall-impact", (4096, 16384))
    out = []
    for v in ("0", "6", "3", "7"):
        monkeypatch.setenv("WB_KSTEP_VARIANT", v)
        sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
        sim.run_steps(3)
        out.append((sim.t, sim.q))
        del sim
    for t, q in out[1:]:
        assert t == out[0][0] and np.array_equal(q, out[0][1])


def test_c3_drop_mass_conservation(torch_cuda):
    from paper_1806_04960_b200.scenarios import build_scenario
    from paper_1806_04960_b200.timestepper import Simulation
    sc = build_scenario("drop", (4096, 4096))
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
    m0 = sim.total_mass(device=True)
    sim.run_steps(100)
    m1 = sim.total_mass(device=True)
    assert abs(m1 - m0) <= 1e-12 * m0
    d = sim.diagnostics()
    assert d["min_alpha"] > 0.0


def test_c2_lake_1000_steps_exact(torch_cuda):
    from paper_1806_04960_b200.scenarios import build_scenario
    from paper_1806_04960_b200.timestepper import Simulation
    sc = build_scenario("lake", (2048, 1024))
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
    sim.run_steps(1000)
    assert np.array_equal(sim.q, sc.q0)

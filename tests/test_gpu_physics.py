"""Physics acceptance checks from SPEC.md:729-738 that run in seconds on the
device (GPU tests): elliptical drop semi-axes (acceptance 3), and the device
depth-averaged velocity diagnostic."""
import math

import numpy as np
import pytest

from paper_1806_04960_b200 import analysis as A
from paper_1806_04960_b200.scenarios import build_scenario

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def drop_run():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1806_04960_b200.timestepper import Simulation
    sc = build_scenario("drop", (200, 200))
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
    out = {}
    for t in (0.0008, 0.0038, 0.0076):
        sim.run_until(t)
        out[t] = (sim.t, sim.q)
    return sc, out


@pytest.mark.parametrize("t", [0.0008, 0.0038, 0.0076])
def test_drop_semi_axes(drop_run, t):
    sc, out = drop_run
    tt, q = out[t]
    assert tt == pytest.approx(t, abs=1e-12)
    g = sc.grid
    a, b, area = A.ellipse_semi_axes(q[..., 3], g.x_centers, g.y_centers, g.dx, g.dy)
    bref = A.drop_reference(t)[1]
    assert abs(b - bref) <= 0.05 * bref, (b, bref)
    assert abs(area - math.pi) <= 0.03 * math.pi, area


def test_depth_averaged_velocity_device(torch_cuda):
    """Device u_bar(x) against the host formula (analysis.py) on a moving
    dambreak: same terms, j-ordered instead of pairwise sums."""
    from paper_1806_04960_b200.analysis import depth_averaged_velocity
    from paper_1806_04960_b200.scenarios import build_scenario
    from paper_1806_04960_b200.timestepper import Simulation
    sc = build_scenario("wall-impact", (300, 160))
    sim = Simulation(sc.grid, sc.params, sc.q0, sc.boundary)
    sim.run_steps(60)
    dev = sim.depth_averaged_velocity()
    host = depth_averaged_velocity(sim.q, sc.grid.mask, sc.grid.dy)
    assert np.abs(host).max() > 0.0
    assert np.allclose(dev, host, rtol=1e-12, atol=1e-12 * np.abs(host).max())

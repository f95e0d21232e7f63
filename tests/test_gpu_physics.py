"""Physics acceptance checks from SPEC.md:729-738 that run in seconds on the
device (GPU tests): elliptical drop semi-axes (acceptance 3)."""
import math

import numpy as np
import pytest

from paper_1806_04960_b200 import analysis as A
from paper_1806_04960_b200.scenarios import build_scenario

pytestmark = pytest.mark.gpu


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

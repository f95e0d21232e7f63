"""Closed-form references (SPEC.md:578-640 examples) -- CPU."""
import math

import numpy as np
import pytest

from paper_1806_04960_b200 import analysis as A


def test_drop_reference():
    a, b = A.drop_reference(0.0076)
    assert b == 1.95 and a == 1.0 / 1.95
    assert A.drop_reference(0.0008)[1] == 1.083
    with pytest.raises(ValueError):
        A.drop_reference(0.001)


def test_jet_surface_branches():
    th = math.radians(60.0)
    ba = np.linspace(1e-3, th - 1e-3, 100)
    bb = np.linspace(th + 1e-3, math.pi / 2 - 1e-3, 100)
    for b in (ba, bb):
        x, y = A.jet_surface_reference(b, th)
        assert np.all(np.isfinite(x)) and np.all(np.isfinite(y))
    # logarithmic asymptotes along the plate as beta -> theta
    ya = A.jet_surface_reference(np.array([th - 1e-2, th - 1e-4]), th)[1]
    assert abs(ya[1]) > abs(ya[0])


def test_jet_pressure():
    q = np.linspace(1e-4, 1 - 1e-4, 2001)
    x, p = A.jet_pressure_reference(q)
    assert np.all(p >= -1e-9)
    assert abs(p.max() - 12500.0) / 12500.0 < 1e-3
    assert p[0] < 1000.0 or p[-1] < 1000.0


def test_weir_profile():
    assert A.weir_profile_reference(0.18) == 0.78
    assert A.weir_profile_reference(0.18 + 0.46) == pytest.approx(0.78 - 0.47 * 0.46)


def test_ritter_and_stoker():
    hl, t, g = 1.4618, 5.0, 9.81
    front = 2 * t * math.sqrt(g * hl)
    assert front == pytest.approx(37.87, abs=0.01)
    x = np.array([-100.0, front - 1e-6, front + 1e-6])
    h, u = A.sw_dambreak_reference(x, t, hl)
    assert h[0] == hl and u[0] == 0.0 and h[1] > 0.0 and h[2] == 0.0
    hm = A.stoker_middle_state(1.5, 0.75)
    cl, cm = math.sqrt(g * 1.5), math.sqrt(g * hm)
    um = 2 * (cl - cm)
    resid = um - (hm - 0.75) * math.sqrt(0.5 * g * (1 / hm + 1 / 0.75))
    assert abs(resid) <= 1e-9
    h, u = A.sw_dambreak_reference(np.linspace(-50, 50, 1001), 10.0, 1.5, 0.75)
    assert np.all(h >= 0.75 - 1e-12) and np.all(h <= 1.5)


def test_depth_average_and_interfaces():
    nx, ny = 20, 30
    q = np.zeros((nx, ny, 5))
    q[..., 0] = 1000.0
    q[..., 3] = 1.0
    q[..., 1] = 1000.0 * 2.5
    ub = A.depth_averaged_velocity(q, np.ones((nx, ny)), 0.1)
    assert np.allclose(ub, 2.5)
    n = 200
    xc = (np.arange(n) + 0.5) * 6.0 / n - 3.0
    X, Y = np.meshgrid(xc, xc, indexing="ij")
    alpha = np.where(X * X + Y * Y <= 1.0, 0.999, 0.001)
    a, b, area = A.ellipse_semi_axes(alpha, xc, xc, 6.0 / n, 6.0 / n)
    assert abs(a - 1.0) < 6.0 / n and abs(b - 1.0) < 6.0 / n
    assert abs(area - math.pi) < 0.05
    segs = A.interface_contour(alpha, xc, xc)
    r = np.hypot(segs[..., 0], segs[..., 1])
    assert np.all(np.abs(r - 1.0) < 6.0 / n)

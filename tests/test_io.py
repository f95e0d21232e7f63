"""Snapshot / time-series IO: bit-exact round trip (CPU)."""
import os
import tempfile
from types import SimpleNamespace

import numpy as np

from paper_1806_04960_b200.io import (TimeSeriesWriter, read_snapshot, write_snapshot)
from paper_1806_04960_b200.scenarios import build_scenario


def test_snapshot_roundtrip_bitexact():
    sc = build_scenario("dambreak-step-wet", (120, 30))
    q = sc.q0.copy()
    rng = np.random.default_rng(0)
    q[..., 1] = rng.standard_normal(q.shape[:2]) * 1e-3   # awkward doubles
    q[..., 0] *= 1.0 + rng.standard_normal(q.shape[:2]) * 1e-12
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "snap.txt")
        write_snapshot(path, q, sc.grid, sc.params, t=0.125, step=7)
        s = read_snapshot(path)
        assert (s.nx, s.ny, s.t, s.step) == (120, 30, 0.125, 7)
        assert (s.x0, s.y0_origin, s.dx, s.dy) == (sc.grid.x0, sc.grid.y0_origin,
                                                   sc.grid.dx, sc.grid.dy)
        assert np.array_equal(s.q, q)
        assert np.array_equal(s.mask, sc.grid.mask)
        fl = sc.grid.mask != 0
        p = sc.params.k0 * (q[..., 0][fl] / q[..., 3][fl] / sc.params.rho0 - 1.0)
        assert np.array_equal(s.p[fl], p)
        assert np.all(s.p[~fl] == 0.0)
        with open(path) as f:
            assert sum(1 for _ in f) == 2 + 120 * 30


def test_timeseries_rows():
    sim = SimpleNamespace(step_count=3, t=0.5, total_mass=lambda: 12.5,
                          stats=SimpleNamespace(dt=0.01, max_rate=45.0, cells_per_second=1e9))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "ts.csv")
        with TimeSeriesWriter(path, extra=("E_rho",)) as w:
            w.row(sim, E_rho=1e-12)
            sim.step_count = 4
            w.row(sim, mass=12.25, E_rho=0.0)
        rows = open(path).read().splitlines()
        assert rows[0] == "step,t,dt,mass,max_rate,cells_per_second,E_rho"
        assert rows[1].split(",")[3] == "12.5" and rows[2].split(",")[3] == "12.25"


"""Snapshot and time-series output (the
format of SPEC.md:670-711, which the reference package does not implement).

Snapshot: a plain-text file.
- One header line:
  ``nx ny x0 y0_origin dx dy t step``
- One record per cell, in i-major order:
  ``i j arho arhou arhov alpha p mask``
- Every float is written with 17 significant digits, so read(write(q)) is
  bit-exact.
- ``p`` is the Tait pressure (0 in solid cells).

Time series: CSV, one row per sampled step with the columns
``step, t, dt, mass, max_rate, cells_per_second`` plus optional
equilibrium errors.

``AsyncSnapshotWriter`` takes a host copy of the state between steps and
formats and writes it on a background thread.  The device keeps stepping
while the file is produced.
"""

import csv
import os
import queue
import threading
from dataclasses import dataclass

import numpy as np

__all__ = ["Snapshot", "write_snapshot", "read_snapshot", "TimeSeriesWriter",
           "AsyncSnapshotWriter"]

_HEADER = ("nx", "ny", "x0", "y0_origin", "dx", "dy", "t", "step")


@dataclass
class Snapshot:
    nx: int
    ny: int
    x0: float
    y0_origin: float
    dx: float
    dy: float
    t: float
    step: int
    q: np.ndarray      # (nx, ny, 5) conserved state, q[..., 4] = y centres
    p: np.ndarray      # (nx, ny) pressure
    mask: np.ndarray   # (nx, ny) uint8


def _pressure(q, mask, params):
    fluid = mask != 0
    rho = np.zeros(q.shape[:2])
    np.divide(q[..., 0], q[..., 3], out=rho, where=fluid)
    p = np.zeros_like(rho)
    ratio = rho / params.rho0
    if params.gamma == 1.0:
        np.multiply(ratio - 1.0, params.k0, out=p, where=fluid)
    else:
        np.multiply(ratio ** params.gamma - 1.0, params.k0, out=p, where=fluid)
    return p


def write_snapshot(path, q, grid, params, t=0.0, step=0):
    """Write the state `q` (nx, ny, 5) of `grid` to `path`."""
    q = np.asarray(q, dtype=np.float64)
    nx, ny = grid.nx, grid.ny
    if q.shape != (nx, ny, 5):
        raise ValueError(f"q must have shape {(nx, ny, 5)}")
    mask = np.asarray(grid.mask, dtype=np.uint8)
    p = _pressure(q, mask, params)
    ii, jj = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    rec = np.column_stack([ii.ravel(), jj.ravel(), q[..., 0].ravel(), q[..., 1].ravel(),
                           q[..., 2].ravel(), q[..., 3].ravel(), p.ravel(), mask.ravel()])
    tmp = path + ".tmp"
    try:
        with open(tmp, "w") as f:
            f.write(" ".join(_HEADER) + "\n")
            f.write(f"{nx} {ny} {grid.x0!r} {grid.y0_origin!r} {grid.dx!r} {grid.dy!r} "
                    f"{float(t)!r} {int(step)}\n")
            np.savetxt(f, rec, fmt=["%d", "%d", "%.17g", "%.17g", "%.17g", "%.17g", "%.17g",
                                    "%d"])
        os.replace(tmp, path)
    except OSError as e:
        raise OSError(f"cannot write snapshot {path}: {e}") from e


def read_snapshot(path):
    """Read a snapshot written by `write_snapshot` (bit-exact)."""
    try:
        with open(path) as f:
            names = f.readline().split()
            vals = f.readline().split()
            data = np.loadtxt(f, dtype=np.float64, ndmin=2)
    except OSError as e:
        raise OSError(f"cannot read snapshot {path}: {e}") from e
    if tuple(names) != _HEADER:
        raise ValueError(f"{path}: not a snapshot (header {names})")
    nx, ny = int(vals[0]), int(vals[1])
    x0, y0o, dx, dy, t = (float(v) for v in vals[2:7])
    step = int(vals[7])
    if data.shape != (nx * ny, 8):
        raise ValueError(f"{path}: expected {nx * ny} records, got {data.shape[0]}")
    q = np.empty((nx, ny, 5))
    for m in range(4):
        q[..., m] = data[:, 2 + m].reshape(nx, ny)
    q[..., 4] = (y0o + (np.arange(ny) + 0.5) * dy)[None, :]
    return Snapshot(nx, ny, x0, y0o, dx, dy, t, step, q,
                    data[:, 6].reshape(nx, ny), data[:, 7].reshape(nx, ny).astype(np.uint8))


class TimeSeriesWriter:
    """CSV rows of per-step diagnostics."""

    COLUMNS = ("step", "t", "dt", "mass", "max_rate", "cells_per_second")

    def __init__(self, path, extra=()):
        self.path = path
        self.extra = tuple(extra)
        self._f = open(path, "w", newline="")
        self._w = csv.writer(self._f)
        self._w.writerow(self.COLUMNS + self.extra)

    def row(self, sim, mass=None, **extra):
        st = sim.stats
        vals = [sim.step_count, repr(float(sim.t)), repr(float(st.dt)),
                repr(float(sim.total_mass() if mass is None else mass)),
                repr(float(st.max_rate)), repr(float(st.cells_per_second))]
        vals += [repr(float(extra[k])) for k in self.extra]
        self._w.writerow(vals)
        self._f.flush()

    def close(self):
        self._f.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class AsyncSnapshotWriter:
    """Write snapshots on a background thread.  ``submit`` copies the state
    to host memory (the only part on the stepping thread), formatting and
    file I/O overlap the next device steps."""

    def __init__(self, grid, params, max_pending=2):
        self.grid, self.params = grid, params
        self._q = queue.Queue(maxsize=max_pending)
        self._errors = []
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()

    def _run(self):
        while True:
            item = self._q.get()
            if item is None:
                return
            path, q, t, step = item
            try:
                write_snapshot(path, q, self.grid, self.params, t, step)
            except Exception as e:  # surfaced on close()
                self._errors.append(e)

    def submit(self, path, sim):
        self._q.put((path, sim.q, sim.t, sim.step_count))

    def close(self):
        self._q.put(None)
        self._th.join()
        if self._errors:
            raise self._errors[0]

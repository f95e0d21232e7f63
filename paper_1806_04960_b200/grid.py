"""Mesh, obstacle mask and boundary conditions (drop-in for ``wbflow.grid``).

API mirror of pkg/src/wbflow/grid.py: ``CartesianGrid`` (21-64), ``build_grid``
(67-96), ``BoundaryCondition`` / ``BoundarySpec`` (99-135), ``ghost_state``
(138-158) and ``enumerate_edges`` (275-279).  The four-colour ``EdgeSet`` of the
reference exists only to make its CPU edge sweeps race-free; the B200 kernels
classify every face on the fly, so here the edge lists are produced by a
vectorised numpy pass (same groups, same order, same bc codes) purely for API
compatibility and tests -- the time loop never touches them.
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError

__all__ = ["CartesianGrid", "build_grid", "BoundaryCondition", "BoundarySpec",
           "ghost_state", "EdgeSet", "enumerate_edges",
           "BC_REFLECTIVE", "BC_TRANSMISSIVE", "BC_INFLOW", "SIDES"]

# boundary codes shared with the CUDA library (kernels.py:29-31)
BC_REFLECTIVE = 1
BC_TRANSMISSIVE = 2
BC_INFLOW = 3
KIND_CODES = {"reflective": BC_REFLECTIVE, "transmissive": BC_TRANSMISSIVE,
              "inflow": BC_INFLOW}
SIDES = ("left", "right", "bottom", "top")


@dataclass(frozen=True)
class CartesianGrid:
    """Cell-centred nx x ny mesh; ``mask`` is uint8 (1 fluid, 0 solid)."""

    nx: int
    ny: int
    x0: float
    y0_origin: float
    dx: float
    dy: float
    mask: np.ndarray

    def __post_init__(self):
        if self.nx < 2 or self.ny < 2:
            raise ConfigError(f"grid must be at least 2x2, got {self.nx}x{self.ny}")
        if not (self.dx > 0.0 and self.dy > 0.0):
            raise ConfigError("grid spacings must be positive")

    # coordinate arrays use numpy's vectorised arithmetic exactly as the
    # reference does (grid.py:40-54), so the device sees identical doubles
    @property
    def x_centers(self):
        return self.x0 + (np.arange(self.nx) + 0.5) * self.dx

    @property
    def y_centers(self):
        return self.y0_origin + (np.arange(self.ny) + 0.5) * self.dy

    @property
    def x_faces(self):
        return self.x0 + np.arange(self.nx + 1) * self.dx

    @property
    def y_faces(self):
        return self.y0_origin + np.arange(self.ny + 1) * self.dy

    @property
    def cell_area(self):
        return self.dx * self.dy

    def is_fluid(self, i, j):
        return self.mask[i, j] != 0

    def fluid_cell_count(self):
        return int(np.count_nonzero(self.mask))


def _snap(lo, hi, origin, h, n, rect):
    a = int(round((lo - origin) / h))
    b = int(round((hi - origin) / h))
    if b <= a:
        b = a + 1
    if a < 0 or b > n:
        raise ConfigError(f"obstacle {rect} lies outside the domain")
    return a, b


def build_grid(domain, resolution, obstacles=()):
    """Mesh over ``domain=(x_min, x_max, y_min, y_max)`` with ``resolution=(nx, ny)``;
    obstacle rectangles are snapped to faces and at least one cell wide
    (grid.py:67-96)."""
    x_min, x_max, y_min, y_max = map(float, domain)
    nx, ny = map(int, resolution)
    if not (x_max > x_min and y_max > y_min):
        raise ConfigError(f"empty domain {domain}")
    if nx < 2 or ny < 2:
        raise ConfigError(f"resolution must be at least 2x2, got {resolution}")
    dx = (x_max - x_min) / nx
    dy = (y_max - y_min) / ny
    mask = np.ones((nx, ny), dtype=np.uint8)
    for rect in obstacles:
        ox0, ox1, oy0, oy1 = map(float, rect)
        i0, i1 = _snap(ox0, ox1, x_min, dx, nx, rect)
        j0, j1 = _snap(oy0, oy1, y_min, dy, ny, rect)
        mask[i0:i1, j0:j1] = 0
    return CartesianGrid(nx, ny, x_min, y_min, dx, dy, mask)


@dataclass(frozen=True)
class BoundaryCondition:
    """One domain side: ``kind`` in {reflective, transmissive, inflow}; inflow
    needs a primitive ``state`` (rho, u, v, alpha, p) and a ``segment`` (lo, hi)
    along the side, outside of which the side is reflective (grid.py:99-123)."""

    kind: str = "reflective"
    state: tuple = None
    segment: tuple = None

    def __post_init__(self):
        if self.kind not in KIND_CODES:
            raise ConfigError(f"unknown boundary kind {self.kind!r}")
        if self.kind == "inflow":
            if self.state is None or self.segment is None:
                raise ConfigError("inflow boundaries need a state and a segment")
            lo, hi = self.segment
            if not hi > lo:
                raise ConfigError(f"empty inflow segment {self.segment}")

    @property
    def code(self):
        return KIND_CODES[self.kind]


@dataclass(frozen=True)
class BoundarySpec:
    left: BoundaryCondition = field(default_factory=BoundaryCondition)
    right: BoundaryCondition = field(default_factory=BoundaryCondition)
    bottom: BoundaryCondition = field(default_factory=BoundaryCondition)
    top: BoundaryCondition = field(default_factory=BoundaryCondition)

    @staticmethod
    def all_reflective():
        return BoundarySpec()

    def side(self, name):
        return getattr(self, name)


def ghost_state(inside, condition, normal):
    """Primitive ghost state across a boundary (API helper, grid.py:138-158).

    Note: the time loop's transmissive ghost resets the density to rho0
    (kernels.py:1082-1084); this helper copies, exactly like the reference."""
    kind = condition.kind if isinstance(condition, BoundaryCondition) else condition
    w = np.array(inside, dtype=float)
    if kind == "reflective":
        w[1 if normal[0] == "x" else 2] *= -1.0
        return w
    if kind == "transmissive":
        return w
    if kind == "inflow":
        return np.array(condition.state, dtype=float)
    raise ConfigError(f"unknown boundary kind {kind!r}")


def _side_modes(cond, coords):
    """Per-face bc code along one side (grid.py:213-220)."""
    if cond.kind == "inflow":
        lo, hi = cond.segment
        inside = (coords >= lo) & (coords <= hi)
        return np.where(inside, BC_INFLOW, BC_REFLECTIVE).astype(np.int64)
    return np.full(coords.shape, KIND_CODES[cond.kind], dtype=np.int64)


def _faces(mask, lo_mode, hi_mode):
    """Faces normal to axis 0 of ``mask`` (shape (n, m)), listed face-index
    major: returns (face index, cross index, bc code) for every face with at
    least one fluid side; codes follow grid.py:223-272."""
    n, m = mask.shape
    fl = np.zeros((n + 2, m), dtype=bool)
    fl[1:-1] = mask != 0
    minus = fl[:-1]          # cell ifc-1 is fluid
    plus = fl[1:]            # cell ifc is fluid
    keep = minus | plus
    mode = np.zeros((n + 1, m), dtype=np.int64)
    only_plus = plus & ~minus
    only_minus = minus & ~plus
    mode[only_plus] = -BC_REFLECTIVE
    mode[only_minus] = BC_REFLECTIVE
    mode[0, only_plus[0]] = -lo_mode[only_plus[0]]
    mode[n, only_minus[n]] = hi_mode[only_minus[n]]
    f, c = np.nonzero(keep)
    return f.astype(np.int64), c.astype(np.int64), mode[f, c].astype(np.int8)


class EdgeSet:
    """Edge lists in the reference's four groups (grid.py:161-210); kept for
    API compatibility (``Simulation.edges``) -- the B200 kernels do not use it."""

    def __init__(self, grid, boundary):
        self.grid = grid
        self.boundary = boundary
        vi, vj, vb = _faces(grid.mask, _side_modes(boundary.left, grid.y_centers),
                            _side_modes(boundary.right, grid.y_centers))
        hj, hi, hb = _faces(grid.mask.T, _side_modes(boundary.bottom, grid.x_centers),
                            _side_modes(boundary.top, grid.x_centers))
        order = np.lexsort((hi, hj))
        hi, hj, hb = hi[order], hj[order], hb[order]
        vodd = vi % 2 == 1
        hodd = hj % 2 == 1
        self.groups = (
            ("vertical-odd", vi[vodd], vj[vodd], vb[vodd]),
            ("vertical-even", vi[~vodd], vj[~vodd], vb[~vodd]),
            ("horizontal-odd", hi[hodd], hj[hodd], hb[hodd]),
            ("horizontal-even", hi[~hodd], hj[~hodd], hb[~hodd]),
        )
        self.vertical = (vi, vj, vb)
        self.horizontal = (hi, hj, hb)

    @property
    def n_edges(self):
        return sum(len(g[1]) for g in self.groups)

    def group_cells(self, group_index):
        name, a, b, bc = self.groups[group_index]
        out = []
        for x, y, m in zip(a.tolist(), b.tolist(), bc.tolist()):
            cells = []
            if name.startswith("vertical"):
                if m >= 0:
                    cells.append((x - 1, y))
                if m <= 0:
                    cells.append((x, y))
            else:
                if m >= 0:
                    cells.append((x, y - 1))
                if m <= 0:
                    cells.append((x, y))
            out.append(cells)
        return out


def enumerate_edges(grid, boundary=None):
    return EdgeSet(grid, boundary if boundary is not None else BoundarySpec())

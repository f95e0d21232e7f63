"""Deterministic scenario / initial-condition builders for the benchmark and
parity configurations (the reference ships none --
SPEC.md:554-659 describes them).

Gravity initial conditions are *detection-consistent* (SURVEY.md App. A.9):
alpha = 1-eps in the liquid and eps in the gas, the column surface level
(y0_i, aeq_i) is detected exactly the way the solver does it
(kernels.py:497-520, sequential sum in j), and the liquid density is
aeq_i * eq_rho(y_j, y0_i) evaluated with libm exp, so that still liquid is
bit-exactly quiet on the first step.
"""

from dataclasses import dataclass
import math

import numpy as np

from .grid import BoundaryCondition, BoundarySpec, build_grid
from .params import ModelParams
from .state import eq_rho_profile

__all__ = ["Scenario", "build_scenario", "detect_columns", "SCENARIOS",
           "column_equilibrium_state", "ColumnEquilibriumIC"]


@dataclass
class ColumnEquilibriumIC:
    """The detection-consistent column-equilibrium initial condition: alpha =
    ``alpha_liq`` in the union of ``boxes`` (closed rectangles (x0, x1, y0, y1)
    of cell centres), ``alpha_gas`` elsewhere; liquid density from each
    column's detected equilibrium, gas (alpha <= 10 eps) at ``gas_rho`` if
    given; at rest.  Built on the host (``host_state``) or directly on the
    device (``Simulation.from_scenario``, C ABI wb_init_column_equilibrium),
    bit for bit the same."""
    boxes: tuple
    alpha_liq: float
    alpha_gas: float
    gas_rho: float = None

    def host_state(self, grid, params, cols=None):
        x, y = _centres(grid, cols)
        liquid = np.zeros(x.shape, dtype=bool)
        for b in self.boxes:
            liquid |= _box(x, y, *b)
        alpha = np.where(liquid, self.alpha_liq, self.alpha_gas)
        return column_equilibrium_state(grid, params, alpha, cols=cols, gas_rho=self.gas_rho)


@dataclass
class Scenario:
    name: str
    grid: object
    params: ModelParams
    boundary: BoundarySpec
    q0: np.ndarray          # (nx, ny, 5) conserved state, reference layout (None if not built)
    t_end: float = None
    col0: int = 0           # first global column held in q0 (x-slab builds)
    ic: ColumnEquilibriumIC = None  # device-buildable initial condition, if any


def detect_columns(alpha, mask, y_faces, dy):
    """(y0s, aeqs) per column, identical to the solver's sequential detection
    (kernels.py:432-453): numpy's add.accumulate is a strictly sequential sum,
    and solid cells contribute an exact +0.0."""
    fluid = mask != 0
    a = np.where(fluid, alpha, 0.0)
    ssum = np.cumsum(a, axis=1)[:, -1]
    any_fluid = fluid.any(axis=1)
    first = np.argmax(fluid, axis=1)
    ylow = np.where(any_fluid, np.asarray(y_faces)[first], y_faces[0])
    aeq = np.where(any_fluid, alpha[np.arange(alpha.shape[0]), first], 1.0)
    return ylow + ssum * dy, aeq


def column_equilibrium_state(grid, params, alpha, u=None, v=None, gas_rho=None, cols=None):
    """Conserved state for a volume-fraction field: liquid density follows
    each column's detected equilibrium aeq*eq_rho(y, y0); gas (alpha <= 10 eps
    when ``gas_rho`` is given) gets rho = gas_rho.  ``alpha`` covers the
    columns ``cols = (lo, hi)`` (all columns by default)."""
    lo, hi = cols if cols is not None else (0, grid.nx)
    nx, ny = hi - lo, grid.ny
    yc = grid.y_centers
    y0s, aeqs = detect_columns(alpha, np.asarray(grid.mask)[lo:hi], grid.y_faces, grid.dy)
    rho_a = np.empty((nx, ny))
    # one libm-exp profile per distinct surface level (few in practice)
    for y0 in np.unique(y0s):
        cols = y0s == y0
        rho_a[cols] = eq_rho_profile(yc, y0, params)[None, :]
    arho = aeqs[:, None] * rho_a
    if gas_rho is not None:
        gas = alpha <= 10.0 * params.epsilon
        arho = np.where(gas, alpha * gas_rho, arho)
    q = np.zeros((nx, ny, 5))
    q[..., 0] = arho
    if u is not None:
        q[..., 1] = arho * u
    if v is not None:
        q[..., 2] = arho * v
    q[..., 3] = alpha
    q[..., 4] = yc[None, :]
    return q


def _centres(grid, cols=None):
    lo, hi = cols if cols is not None else (0, grid.nx)
    return np.meshgrid(grid.x_centers[lo:hi], grid.y_centers, indexing="ij")


def _box(x, y, x0, x1, y0, y1):
    return (x >= x0) & (x <= x1) & (y >= y0) & (y <= y1)


def _liquid_state(grid, params, liquid, u=None, v=None):
    """Conserved state for a g = 0 case: rho = rho0 everywhere, alpha =
    1-eps in the liquid (velocity (u, v) there) and eps in the gas (at rest)."""
    eps = params.epsilon
    alpha = np.where(liquid, 1.0 - eps, eps)
    q = np.zeros(alpha.shape + (5,))
    q[..., 0] = alpha * params.rho0
    if u is not None:
        q[..., 1] = np.where(liquid, q[..., 0] * u, 0.0)
    if v is not None:
        q[..., 2] = np.where(liquid, q[..., 0] * v, 0.0)
    q[..., 3] = alpha
    q[..., 4] = grid.y_centers[None, :]
    return q


def _dambreak_ic(params, regions, gas_rho=None):
    """Dambreak with one or several liquid rectangles (gas at gas_rho, default rho0)."""
    eps = params.epsilon
    return ColumnEquilibriumIC(tuple(tuple(float(v) for v in r) for r in regions), 1.0 - eps,
                               eps, params.rho0 if gas_rho is None else gas_rho)


def _state(ic, grid, params, cols, host):
    return ic.host_state(grid, params, cols) if host else None


def _lake(name, res, obstacles, perturb_seed=None, host=True):
    params = ModelParams(k0=2.78e5)
    grid = build_grid((-0.5, 0.5, 0.0, 1.0), res, obstacles)
    ic = ColumnEquilibriumIC((), 1.0, 1.0, None)  # alpha = 1 everywhere
    if perturb_seed is None:
        return Scenario(name, grid, params, BoundarySpec(), _state(ic, grid, params, None, host),
                        ic=ic)
    q = ic.host_state(grid, params)
    rng = np.random.default_rng(perturb_seed)
    kx, ky = rng.integers(1, 4, size=2)
    phi = rng.uniform(0.0, 2.0 * math.pi)
    x, y = _centres(grid)
    rho = q[..., 0] * (1.0 + 1e-3 * np.sin(2 * math.pi * kx * x + phi)
                       * np.cos(2 * math.pi * ky * y))
    u = 1e-2 * np.cos(2 * math.pi * ky * y)
    v = 1e-2 * np.sin(2 * math.pi * kx * x)
    q[..., 0] = rho
    q[..., 1] = rho * u
    q[..., 2] = rho * v
    return Scenario(name, grid, params, BoundarySpec(), q)


LAKE_OBSTACLES = ((-0.25, 0.25, 0.0, 0.33), (0.30, 0.40, 0.0, 0.60),
                  (-0.45, -0.35, 0.0, 0.17))


def build_scenario(name, resolution=None, seed=0, columns=None, host_state=True):
    """Build one named configuration.

    * ``dambreak-dry``  -- C1, [-50,50]x[0,4], liquid [-50,0]x[0,1.4618], k0 6.37e5
      (PAPER.md:1089-1094); reflective L/R/bottom, transmissive top.
    * ``lake``          -- C2, lake at rest with alpha = 1 over three bottom
      obstacles, k0 2.78e5 (PAPER.md:849-851 plus two survey obstacles).
    * ``equilibrium-obstacle`` -- the paper's single-obstacle lake.
    * ``perturbed-lake`` -- C2 geometry with a seeded smooth perturbation.
    * ``drop``          -- C3, [-3,3]^2, g = 0, k0 2.25e9, u = (-100x, 100y) in r<1.
    * ``weir``          -- C4, [-7.5,7.5]x[0,2.1], strip [0,dx]x[0,0.7], liquid
      [-7.5,0]x[0,1.5], k0 6.54e5.
    * ``wall-impact``   -- C5, [0,3.2]x[0,1.8], liquid [0,1.2]x[0,0.6], k0 2.62e5,
      transmissive top.
    * ``jet``           -- small inflow case (inflow segment on the left side,
      transmissive right/top) that exercises the inflow ghost.
    * ``dambreak-wet`` / ``dambreak-step-dry`` / ``dambreak-step-wet`` -- PAPER.md
      section 5.6.2-5.6.4 (wet bed, 0.2 bottom step).
    * ``equilibrium-flat`` -- the paper's flat-bottom lake at rest (100x100).
    * ``spinning-square`` / ``jet-plate`` -- PAPER.md sections 5.3 / 5.4 (g = 0).
    * ``tait7``         -- a gamma = 7 dambreak (pow() path; parity by tolerance).

    ``columns=(lo, hi)`` builds only those columns of q0 (x-slab of a
    multi-GPU run; supported by the dambreak-type scenarios); the grid is
    always the global one.  The column-equilibrium scenarios (dambreaks, weir,
    wall-impact, unperturbed lakes) carry ``ic``; with ``host_state=False``
    their q0 is not built on the host (``Simulation.from_scenario`` builds it
    on the device).
    """
    if columns is not None and name not in ("dambreak-dry", "weir", "wall-impact",
                                            "dambreak-wet", "dambreak-step-dry",
                                            "dambreak-step-wet"):
        sc = build_scenario(name, resolution, seed)
        lo, hi = columns
        sc.q0 = np.ascontiguousarray(sc.q0[lo:hi])
        sc.col0 = lo
        return sc
    cols = columns
    if name == "dambreak-dry":
        res = resolution or (200, 100)
        params = ModelParams(k0=6.37e5)
        grid = build_grid((-50.0, 50.0, 0.0, 4.0), res)
        ic = _dambreak_ic(params, [(-50.0, 0.0, 0.0, 1.4618)])
        bnd = BoundarySpec(top=BoundaryCondition("transmissive"))
        return Scenario(name, grid, params, bnd, _state(ic, grid, params, cols, host_state),
                        col0=cols[0] if cols else 0, ic=ic)
    if name in ("dambreak-wet", "dambreak-step-dry", "dambreak-step-wet"):
        # PAPER.md section 5.6.2-5.6.4 (Omega = [-50,50]x[0,4], step [0,50]x[0,0.2])
        res = resolution or (4000, 400)
        wet = name != "dambreak-step-dry"
        params = ModelParams(k0=6.54e5 if wet else 6.37e5)
        step = name.startswith("dambreak-step")
        grid = build_grid((-50.0, 50.0, 0.0, 4.0), res,
                          [(0.0, 50.0, 0.0, 0.2)] if step else ())
        if name == "dambreak-wet":
            regions = [(-50.0, 0.0, 0.0, 1.5), (0.0, 50.0, 0.0, 0.75)]
        elif name == "dambreak-step-dry":
            regions = [(-50.0, 0.0, 0.0, 0.4618)]
        else:
            regions = [(-50.0, 0.0, 0.0, 0.4618), (0.0, 50.0, 0.2, 0.50873)]
        ic = _dambreak_ic(params, regions)
        bnd = BoundarySpec(top=BoundaryCondition("transmissive"))
        return Scenario(name, grid, params, bnd, _state(ic, grid, params, cols, host_state),
                        col0=cols[0] if cols else 0, ic=ic)
    if name == "equilibrium-flat":
        return _lake(name, resolution or (100, 100), (), host=host_state)
    if name == "spinning-square":
        # PAPER.md section 5.3: [-5,5]^2, square [-1,1]^2, u = (2 pi y, -2 pi x), k0 8.78e5, g 0
        res = resolution or (850, 850)
        params = ModelParams(k0=8.78e5, g=0.0)
        grid = build_grid((-5.0, 5.0, -5.0, 5.0), res)
        x, y = _centres(grid)
        liquid = _box(x, y, -1.0, 1.0, -1.0, 1.0)
        q = _liquid_state(grid, params, liquid, 2.0 * math.pi * y, -2.0 * math.pi * x)
        return Scenario(name, grid, params, BoundarySpec(), q)
    if name == "jet-plate":
        # PAPER.md section 5.4: [-6,8]x[0,10], strip -2 <= y - sqrt(3) x <= 0,
        # |u| = 5 along the jet towards the plate y = 0, k0 2.78e5, g 0
        res = resolution or (500, 350)
        params = ModelParams(k0=2.78e5, g=0.0)
        grid = build_grid((-6.0, 8.0, 0.0, 10.0), res)
        x, y = _centres(grid)
        s3 = math.sqrt(3.0)
        liquid = (y - s3 * x <= 0.0) & (y - s3 * x >= -2.0)
        q = _liquid_state(grid, params, liquid, -5.0 * 0.5, -5.0 * s3 / 2.0)
        bnd = BoundarySpec(left=BoundaryCondition("transmissive"),
                           right=BoundaryCondition("transmissive"),
                           top=BoundaryCondition("transmissive"))
        return Scenario(name, grid, params, bnd, q)
    if name == "lake":
        return _lake(name, resolution or (2048, 1024), LAKE_OBSTACLES, host=host_state)
    if name == "equilibrium-obstacle":
        return _lake(name, resolution or (100, 100), LAKE_OBSTACLES[:1], host=host_state)
    if name == "perturbed-lake":
        return _lake(name, resolution or (128, 128), LAKE_OBSTACLES, perturb_seed=seed)
    if name == "drop":
        res = resolution or (4096, 4096)
        params = ModelParams(k0=2.25e9, g=0.0)
        grid = build_grid((-3.0, 3.0, -3.0, 3.0), res)
        x, y = _centres(grid)
        inside = x * x + y * y <= 1.0
        eps = params.epsilon
        alpha = np.where(inside, 1.0 - eps, eps)
        rho = params.rho0
        q = np.zeros((grid.nx, grid.ny, 5))
        q[..., 0] = alpha * rho
        q[..., 1] = np.where(inside, q[..., 0] * (-100.0 * x), 0.0)
        q[..., 2] = np.where(inside, q[..., 0] * (100.0 * y), 0.0)
        q[..., 3] = alpha
        q[..., 4] = grid.y_centers[None, :]
        return Scenario(name, grid, params, BoundarySpec(), q)
    if name == "weir":
        res = resolution or (16384, 8192)
        params = ModelParams(k0=6.54e5)
        dx = 15.0 / res[0]
        grid = build_grid((-7.5, 7.5, 0.0, 2.1), res, [(0.0, dx, 0.0, 0.7)])
        ic = _dambreak_ic(params, [(-7.5, 0.0, 0.0, 1.5)])
        return Scenario(name, grid, params, BoundarySpec(),
                        _state(ic, grid, params, cols, host_state),
                        col0=cols[0] if cols else 0, ic=ic)
    if name == "wall-impact":
        res = resolution or (32768, 16384)
        params = ModelParams(k0=2.62e5)
        grid = build_grid((0.0, 3.2, 0.0, 1.8), res)
        ic = _dambreak_ic(params, [(0.0, 1.2, 0.0, 0.6)])
        bnd = BoundarySpec(top=BoundaryCondition("transmissive"))
        return Scenario(name, grid, params, bnd, _state(ic, grid, params, cols, host_state),
                        col0=cols[0] if cols else 0, ic=ic)
    if name == "jet":
        res = resolution or (96, 64)
        params = ModelParams(k0=2.78e5, g=9.81)
        grid = build_grid((0.0, 3.0, 0.0, 2.0), res, [(1.8, 2.1, 0.0, 0.9)])
        q = _dambreak_ic(params, [(0.0, 0.6, 0.0, 0.5)]).host_state(grid, params)
        eps = params.epsilon
        state = (params.rho0, 2.0, 0.0, 1.0 - eps, 0.0)
        bnd = BoundarySpec(left=BoundaryCondition("inflow", state, (0.2, 0.6)),
                           right=BoundaryCondition("transmissive"),
                           top=BoundaryCondition("transmissive"))
        return Scenario(name, grid, params, bnd, q)
    if name == "tait7":
        res = resolution or (64, 32)
        params = ModelParams(k0=3.0e5, gamma=7.0)
        grid = build_grid((-4.0, 4.0, 0.0, 2.0), res)
        eps = params.epsilon
        x, y = _centres(grid)
        alpha = np.where(_box(x, y, -4.0, 0.0, 0.0, 1.0), 1.0 - eps, eps)
        rho = params.rho0
        q = np.zeros((grid.nx, grid.ny, 5))
        q[..., 0] = alpha * rho
        q[..., 3] = alpha
        q[..., 4] = grid.y_centers[None, :]
        return Scenario(name, grid, params, BoundarySpec(), q)
    raise ValueError(f"unknown scenario {name!r}")


SCENARIOS = ("dambreak-dry", "dambreak-wet", "dambreak-step-dry", "dambreak-step-wet", "lake",
             "equilibrium-flat", "equilibrium-obstacle", "perturbed-lake", "drop",
             "spinning-square", "jet-plate", "weir", "wall-impact", "jet", "tait7")

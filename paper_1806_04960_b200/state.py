"""Conserved/primitive conversions and the gamma=1 equilibrium family
(subset of ``wbflow.state``, pkg/src/wbflow/state.py:57-122) needed by the
drop-in driver and the scenario builders.

``eq_rho`` evaluates rho0*exp(-(g rho0/k0)(y - y0)) with the C library's
``exp`` (Python's ``math.exp``), which is what the reference's Numba kernels
call (kernels.py:53-55); numpy's SIMD exp differs by 1 ulp on ~5% of inputs
and would break the bit-exact quiet test of still water.
"""

import math

import numpy as np

from .errors import UnsupportedConfigurationError

__all__ = ["tait_pressure", "sound_speed", "cons_to_prim", "prim_to_cons",
           "eq_rho", "eq_rho_profile", "EquilibriumProfile"]


def tait_pressure(rho, params):
    """k0((rho/rho0)^gamma - 1) (kernels.py:38-43)."""
    rho = np.asarray(rho, dtype=np.float64)
    if np.any(rho <= 0.0):
        raise ValueError(f"density must be positive, got {rho}")
    ratio = rho / params.rho0
    out = params.k0 * (ratio - 1.0) if params.gamma == 1.0 else \
        params.k0 * (ratio ** params.gamma - 1.0)
    return float(out) if out.ndim == 0 else out


def sound_speed(rho, params):
    rho = np.asarray(rho, dtype=np.float64)
    if np.any(rho <= 0.0):
        raise ValueError(f"density must be positive, got {rho}")
    if params.gamma == 1.0:
        c2 = np.full(rho.shape, params.k0 / params.rho0)
    else:
        c2 = params.gamma * params.k0 / params.rho0 * (rho / params.rho0) ** (params.gamma - 1.0)
    c = np.sqrt(c2)
    return float(c) if c.ndim == 0 else c


def cons_to_prim(q, params, cell=None):
    """(a rho, a rho u, a rho v, a, y) -> (rho, u, v, alpha, p) (state.py:57-66)."""
    q = np.asarray(q, dtype=np.float64)
    if not (q[0] > 0.0 and q[3] > 0.0):
        where = f" at cell {cell}" if cell is not None else ""
        raise ValueError(f"corrupted state{where}: a*rho = {q[0]}, alpha = {q[3]}")
    rho = q[0] / q[3]
    return np.array([rho, q[1] / q[0], q[2] / q[0], q[3], tait_pressure(rho, params)])


def prim_to_cons(w, y):
    """(rho, u, v, alpha, p), height -> conserved 5-vector (state.py:69-73)."""
    w = np.asarray(w, dtype=np.float64)
    ar = w[3] * w[0]
    return np.array([ar, ar * w[1], ar * w[2], w[3], float(y)])


def eq_rho(y, y0, params):
    """Scalar exponential equilibrium density (kernels.py:53-55), libm exp."""
    return params.rho0 * math.exp(-(params.g * params.rho0 / params.k0) * (y - y0))


def eq_rho_profile(ys, y0, params):
    """eq_rho over an array of heights for one surface level y0."""
    coef = -(params.g * params.rho0 / params.k0)
    r0 = params.rho0
    return np.fromiter((r0 * math.exp(coef * (y - y0)) for y in np.asarray(ys).tolist()),
                       dtype=np.float64, count=len(ys))


class EquilibriumProfile:
    """Water at rest, gamma = 1 closed form (state.py:76-117)."""

    def __init__(self, y0, params, alpha_eq=1.0):
        if params.gamma != 1.0:
            raise UnsupportedConfigurationError(
                f"closed-form equilibria require gamma = 1, got {params.gamma}")
        if not 0.0 < alpha_eq <= 1.0:
            raise ValueError(f"alpha_eq must lie in (0, 1], got {alpha_eq}")
        self.y0, self.params, self.alpha_eq = y0, params, alpha_eq

    def rho(self, y):
        if np.isscalar(y):
            return eq_rho(float(y), self.y0, self.params)
        y = np.asarray(y, dtype=np.float64)
        return eq_rho_profile(y.ravel(), self.y0, self.params).reshape(y.shape)

    def pressure(self, y):
        return tait_pressure(self.rho(y), self.params)

    def primitive(self, y):
        r = self.rho(y)
        return np.array([r, 0.0, 0.0, self.alpha_eq, tait_pressure(r, self.params)])

    def conserved(self, y):
        return prim_to_cons(self.primitive(y), y)

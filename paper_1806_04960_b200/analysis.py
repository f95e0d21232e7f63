"""Closed-form references and analysis helpers for the paper's test cases
(SPEC.md:578-640 -- the reference package does
not implement them).  Host-side numpy; none of this is on the time-stepping
path.

* ``drop_reference(t)``        -- elliptical drop semi-axes
* ``jet_surface_reference``    -- free streamline of the oblique jet
                                  (PAPER.md eq. Jet_freesurface_exact_A/B)
* ``jet_pressure_reference``   -- plate pressure (PAPER.md eq. jet_pressure_exact)
* ``weir_profile_reference``   -- overtopping nappe (PAPER.md eq. OverToppingProfile)
* ``sw_dambreak_reference``    -- Ritter (dry) / Stoker (wet) shallow-water solutions
* ``depth_averaged_velocity``  -- u_bar(x) = sum(u alpha dy) / sum(alpha dy)
* ``interface_contour``        -- marching-squares alpha iso-line
* ``ellipse_semi_axes``        -- semi-axes of the alpha >= level region by moments
"""

import math

import numpy as np

__all__ = ["drop_reference", "jet_surface_reference", "jet_pressure_reference",
           "weir_profile_reference", "sw_dambreak_reference", "stoker_middle_state",
           "depth_averaged_velocity", "interface_contour", "ellipse_semi_axes"]

_DROP = {0.0008: 1.083, 0.0038: 1.44, 0.0076: 1.95}


def drop_reference(t):
    """(a, b) = (1/b, b) of the elliptical drop at the paper's tabulated times."""
    for tt, b in _DROP.items():
        if abs(t - tt) <= 1e-12:
            return 1.0 / b, b
    raise ValueError(f"untabulated drop time {t}; available {sorted(_DROP)}")


def jet_surface_reference(beta, theta=math.radians(60.0)):
    """Parametric free surface (x, y) of the jet for parameter beta (radians):
    branch A for 0 < beta < theta, branch B for theta < beta < pi/2."""
    beta = np.asarray(beta, dtype=np.float64)
    if np.any(beta <= 0.0) or np.any(beta >= math.pi / 2) or np.any(beta == theta):
        raise ValueError("beta must lie in (0, theta) or (theta, pi/2)")
    st, ct = math.sin(theta), math.cos(theta)
    a = beta < theta
    lt = np.log(np.tan(0.5 * beta))
    lh = np.log(0.5 * np.sin(beta))
    sp = np.sin(0.5 * (theta + beta))
    sm = np.where(a, np.sin(0.5 * (theta - beta)), np.sin(0.5 * (beta - theta)))
    base = np.where(a, (theta - math.pi) * st, theta * st)
    x = (base + lt + ct * (lh - np.log(sp * sm))) / math.pi
    y0 = np.where(a, 0.5 * math.pi * (1.0 + ct), 0.5 * math.pi * (1.0 - ct))
    y = (y0 + st * (np.log(sp) - np.log(sm))) / math.pi
    return x, y


def jet_pressure_reference(q, theta=math.radians(60.0), rho0=1000.0, u_mag=5.0, const=0.0):
    """Plate pressure (x(q), p(q)) of the oblique jet, 0 < q < 1 (Bernoulli)."""
    q = np.asarray(q, dtype=np.float64)
    if np.any(q <= 0.0) or np.any(q >= 1.0):
        raise ValueError("q must lie in (0, 1)")
    st, ct = math.sin(theta), math.cos(theta)
    x = ((1.0 + ct) * np.log1p(q) - (1.0 - ct) * np.log1p(-q)) / (2.0 * math.pi) \
        + st * np.arcsin(q) / math.pi + const
    with np.errstate(divide="ignore", invalid="ignore"):
        s = (-(1.0 - q * ct) + np.sqrt(1.0 - q * q) * st) / (q - ct)
    s = np.where(np.isfinite(s), s, 0.0)  # q = cos(theta): removable singularity, s -> 0
    p = 0.5 * rho0 * u_mag * u_mag * (1.0 - s * s)
    return x, p


def weir_profile_reference(x, x_m=0.18, y_m=0.78, h0bar=0.46):
    """Lower nappe y(x) = y_m - 0.47 h0 ((x - x_m)/h0)^1.85, x >= x_m."""
    x = np.asarray(x, dtype=np.float64)
    if np.any(x < x_m):
        raise ValueError("x must be >= x_m")
    return y_m - 0.47 * h0bar * ((x - x_m) / h0bar) ** 1.85


def stoker_middle_state(hl, hr, g=9.81, tol=1e-12):
    """Middle depth h_m of the wet-bed dambreak (rarefaction + shock) by
    bisection on u_rarefaction(h) = u_shock(h)."""
    if not hl > hr > 0.0:
        raise ValueError("need hl > hr > 0")
    cl = math.sqrt(g * hl)

    def f(h):
        u_raref = 2.0 * (cl - math.sqrt(g * h))
        u_shock = (h - hr) * math.sqrt(0.5 * g * (1.0 / h + 1.0 / hr))
        return u_raref - u_shock

    lo, hi = hr, hl
    while hi - lo > tol * hl:
        mid = 0.5 * (lo + hi)
        if f(mid) > 0.0:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def sw_dambreak_reference(x, t, hl, hr=0.0, g=9.81, x0=0.0):
    """Shallow-water dambreak depth h(x, t) and velocity u(x, t): Ritter for a
    dry bed (hr = 0), Stoker (rarefaction, middle state, bore) for hr > 0."""
    x = np.asarray(x, dtype=np.float64) - x0
    if t <= 0.0:
        raise ValueError("t must be positive")
    cl = math.sqrt(g * hl)
    h = np.where(x < 0.0, hl, hr).astype(np.float64)
    u = np.zeros_like(h)
    if hr == 0.0:
        fan = (x >= -cl * t) & (x <= 2.0 * cl * t)
        h = np.where(fan, (2.0 * cl - x / t) ** 2 / (9.0 * g), np.where(x < -cl * t, hl, 0.0))
        u = np.where(fan, 2.0 / 3.0 * (cl + x / t), 0.0)
        return h, u
    hm = stoker_middle_state(hl, hr, g)
    cm = math.sqrt(g * hm)
    um = 2.0 * (cl - cm)
    s = hm * um / (hm - hr)  # bore speed (mass jump condition)
    fan = (x >= -cl * t) & (x <= (um - cm) * t)
    mid = (x > (um - cm) * t) & (x <= s * t)
    h = np.where(x < -cl * t, hl, h)
    h = np.where(fan, (2.0 * cl - x / t) ** 2 / (9.0 * g), h)
    u = np.where(fan, 2.0 / 3.0 * (cl + x / t), u)
    h = np.where(mid, hm, h)
    u = np.where(mid, um, u)
    h = np.where(x > s * t, hr, h)
    return h, u


def depth_averaged_velocity(q, mask, dy):
    """u_bar per column = sum(u alpha dy) / sum(alpha dy) over fluid cells."""
    fluid = np.asarray(mask) != 0
    alpha = np.where(fluid, q[..., 3], 0.0)
    u = np.zeros_like(alpha)
    np.divide(q[..., 1], q[..., 0], out=u, where=fluid)
    num = np.sum(u * alpha * dy, axis=1)
    den = np.sum(alpha * dy, axis=1)
    return np.divide(num, den, out=np.zeros_like(num), where=den > 0)


def interface_contour(alpha, xc, yc, level=0.5):
    """Marching-squares segments of the alpha = level iso-line on the cell
    centres: array (n, 2, 2) of segment end points."""
    a = np.asarray(alpha, dtype=np.float64)
    segs = []
    nx, ny = a.shape

    def interp(p0, p1, v0, v1):
        t = (level - v0) / (v1 - v0)
        return (p0[0] + t * (p1[0] - p0[0]), p0[1] + t * (p1[1] - p0[1]))

    for i in range(nx - 1):
        for j in range(ny - 1):
            v = (a[i, j], a[i + 1, j], a[i + 1, j + 1], a[i, j + 1])
            p = ((xc[i], yc[j]), (xc[i + 1], yc[j]), (xc[i + 1], yc[j + 1]), (xc[i], yc[j + 1]))
            pts = []
            for k in range(4):
                v0, v1 = v[k], v[(k + 1) % 4]
                if (v0 - level) * (v1 - level) < 0.0:
                    pts.append(interp(p[k], p[(k + 1) % 4], v0, v1))
            for k in range(0, len(pts) - 1, 2):
                segs.append((pts[k], pts[k + 1]))
    return np.array(segs, dtype=np.float64).reshape(-1, 2, 2)


def ellipse_semi_axes(alpha, xc, yc, dx, dy, level=0.5):
    """Semi-axes (a <= b) of the region alpha >= level from its second moments
    (for an ellipse, the covariance eigenvalues are a^2/4 and b^2/4)."""
    inside = np.asarray(alpha) >= level
    x, y = np.meshgrid(xc, yc, indexing="ij")
    w = inside.astype(np.float64) * dx * dy
    area = w.sum()
    if area <= 0.0:
        raise ValueError("empty region")
    mx, my = (w * x).sum() / area, (w * y).sum() / area
    cxx = (w * (x - mx) ** 2).sum() / area
    cyy = (w * (y - my) ** 2).sum() / area
    cxy = (w * (x - mx) * (y - my)).sum() / area
    ev = np.linalg.eigvalsh(np.array([[cxx, cxy], [cxy, cyy]]))
    a, b = 2.0 * np.sqrt(np.maximum(ev, 0.0))
    return float(a), float(b), float(area)

"""Drop-in ``Simulation`` for the reference's time stepper, backed by B200 kernels.

Mirrors pkg/src/wbflow/timestepper.py: the constructor signature
``Simulation(grid, params, q0, boundary=None, cfl=0.45, workers=1)``
(timestepper.py:51), ``advance`` / ``run_until`` / ``max_rate`` / ``detect`` /
``total_mass`` / ``primitive_fields``, the ``t`` / ``step_count`` / ``stats``
attributes, the module functions ``set_workers`` / ``compute_dt`` /
``advance_step`` / ``total_mass``, and the error contract (same
``SimulationError`` messages, step and cell; a failed step is not committed).

The state lives on the GPU in SoA planes; ``sim.q`` is downloaded lazily in
the reference layout (nx, ny, 5) into a cached host mirror.  As in the
reference, where ``q`` is the live state array (timestepper.py:68, 209),
in-place writes such as ``sim.q[i, j, 0] *= 1.001`` take effect: a mirror
handed out by ``sim.q`` is uploaded again before the next device operation
(step, rate, detection, diagnostics).  ``sim.q_next`` is a read-only copy.  The reference's per-step work arrays
(fW..fN, vol, psi, quiet, DW..DN, rhoE_c, rhoE_fy) are produced only when the
simulation is created with ``debug=True`` -- the fused kernel then also
stores them -- because the production path never materialises them.
"""

import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import WbConfig, WbError, WbStatus, WbStageArrays, check, dptr, u8ptr
from .errors import SimulationError, UnsupportedConfigurationError
from .grid import BoundarySpec, EdgeSet, KIND_CODES, SIDES

__all__ = ["Simulation", "set_workers", "compute_dt", "advance_step", "total_mass",
           "StepStats"]

_MESSAGES = {
    _lib.ERR_CELL_STATE: "non-admissible cell state",
    _lib.ERR_FACE: "non-admissible reconstructed face state",
    _lib.ERR_MASS: "negative mass or volume fraction after update",
}


def set_workers(n):
    """API compatibility with timestepper.py:27-30.  The device path has no
    CPU worker pool and its results do not depend on any launch parameter."""
    return max(1, int(n))


@dataclass
class StepStats:
    dt: float = 0.0
    max_rate: float = 0.0
    mass: float = 0.0
    cells_per_second: float = 0.0


def _inflow_conserved(cond):
    if cond.kind != "inflow":
        return (0.0, 0.0, 0.0, 0.0)
    w = np.asarray(cond.state, dtype=np.float64)
    ar = w[3] * w[0]  # prim_to_cons (state.py:69-73)
    return (float(ar), float(ar * w[1]), float(ar * w[2]), float(w[3]))


def make_config(grid, params, boundary, cfl, i_begin=0, i_end=None, device=0,
                rows_per_block=0):
    c = WbConfig()
    c.nx, c.ny = grid.nx, grid.ny
    c.i_begin = i_begin
    c.i_end = grid.nx if i_end is None else i_end
    c.dx, c.dy = float(grid.dx), float(grid.dy)
    c.k0, c.rho0, c.gamma = float(params.k0), float(params.rho0), float(params.gamma)
    c.g, c.epsilon = float(params.g), float(params.epsilon)
    c.cfl = float(cfl)
    for s, name in enumerate(SIDES):
        cond = boundary.side(name)
        c.bc_kind[s] = KIND_CODES[cond.kind]
        if cond.kind == "inflow":
            c.inflow_seg[s][0], c.inflow_seg[s][1] = (float(v) for v in cond.segment)
        for m, v in enumerate(_inflow_conserved(cond)):
            c.inflow_q[s][m] = v
    c.device = int(device)
    c.rows_per_block = int(rows_per_block)
    return c


class Simulation:
    """Device-resident double-buffered simulation (timestepper.py:48-103)."""

    def __init__(self, grid, params, q0, boundary=None, cfl=0.45, workers=1, device=0,
                 debug=False, rows_per_block=0, device_ic=None):
        if not 0.0 < cfl < 1.0:
            raise SimulationError(f"cfl must lie in (0, 1), got {cfl}")
        self.grid = grid
        self.params = params
        self.boundary = boundary if boundary is not None else BoundarySpec()
        self.cfl = float(cfl)
        self.stats = StepStats()
        self.debug = bool(debug)
        self.device = int(device)
        set_workers(workers)
        nx, ny = grid.nx, grid.ny
        if q0 is None and device_ic is None:
            raise SimulationError("q0 is required (or a device-buildable initial condition)")
        if q0 is not None:
            q0 = np.asarray(q0, dtype=np.float64)
            if q0.shape != (nx, ny, 5):
                raise SimulationError(f"q0 must have shape {(nx, ny, 5)}, got {q0.shape}")
        self._L = _lib.load()
        self._fluid = np.asarray(grid.mask) != 0
        # flat indices of the solid cells (usually none): a boolean-mask gather
        # over the whole grid would cost ~0.1 s per transfer at 4096 x 16384
        self._solid_flat = np.flatnonzero(~self._fluid.ravel())
        self._n_fluid = int(np.count_nonzero(self._fluid))
        self._ycent = np.ascontiguousarray(grid.y_centers, dtype=np.float64)
        self._yfaces = np.ascontiguousarray(grid.y_faces, dtype=np.float64)
        self._xcent = np.ascontiguousarray(grid.x_centers, dtype=np.float64)
        mask = np.ascontiguousarray(grid.mask, dtype=np.uint8)
        cfg = make_config(grid, params, self.boundary, cfl, device=device,
                          rows_per_block=rows_per_block)
        h = ctypes.c_void_p()
        check(self._L.wb_create(ctypes.byref(cfg), u8ptr(mask), dptr(self._xcent),
                                dptr(self._ycent), dptr(self._yfaces), ctypes.byref(h)),
              "wb_create")
        self._h = h
        self._t = 0.0
        self._step = 0
        self._edges = None
        self._qh = None           # cached host mirror of the current state
        self._qh_exposed = False  # handed out by the q property (may be written)
        if q0 is not None:
            self._set_q(q0)
        else:
            self._init_on_device(device_ic)
        if self.debug:
            for name in ("fW", "fE", "fS", "fN", "vol", "psi", "DW", "DE", "DS", "DN"):
                setattr(self, name, np.zeros((nx, ny, 5)))
            self.quiet = np.zeros((nx, ny), dtype=np.uint8)
            self.rhoE_c = np.zeros((nx, ny))
            self.rhoE_fy = np.zeros((nx, ny + 1))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._L.wb_destroy(h)
            except Exception:
                pass
            self._h = None

    # ---- state transfer ---------------------------------------------------
    def _set_q(self, q):
        self._qh = None
        self._qh_exposed = False
        q = np.ascontiguousarray(q, dtype=np.float64)
        # solid cells never change (kernels.py:1241-1244); keep their host
        # values so that sim.q returns them bit-exactly
        self._solid_q = q.reshape(-1, 5)[self._solid_flat].copy()
        bi, bj = ctypes.c_int32(-1), ctypes.c_int32(-1)
        rc = self._L.wb_set_state(self._h, q.ctypes.data_as(ctypes.c_void_p), 0,
                                  self.grid.nx, 0, ctypes.byref(bi), ctypes.byref(bj))
        if rc == _lib.WB_E_HEIGHT:
            raise UnsupportedConfigurationError(
                "q0[..., 4] must equal grid.y_centers in fluid cells (the height "
                f"component is derived on the device); cell ({bi.value}, {bj.value}) differs")
        check(rc, "wb_set_state")

    def _get_q(self, which=0, out=None):
        nx, ny = self.grid.nx, self.grid.ny
        q = out if out is not None else np.empty((nx, ny, 5))
        check(self._L.wb_get_state_buf(self._h, q.ctypes.data_as(ctypes.c_void_p), which, 0),
              "wb_get_state")
        if self._solid_flat.size and self._solid_q is not None:
            q.reshape(-1, 5)[self._solid_flat] = self._solid_q
        return q

    @classmethod
    def from_scenario(cls, sc, cfl=0.45, device=0, debug=False, rows_per_block=0,
                      device_ic=True):
        """Simulation of a ``scenarios.Scenario``.  A column-equilibrium initial
        condition (``sc.ic``) is built directly on the device -- no host q0,
        no upload (``build_scenario(..., host_state=False)`` skips the host
        build too); anything else uploads ``sc.q0``."""
        if device_ic and sc.ic is not None:
            return cls(sc.grid, sc.params, None, sc.boundary, cfl=cfl, device=device,
                       debug=debug, rows_per_block=rows_per_block, device_ic=sc.ic)
        if sc.q0 is None:
            raise SimulationError(f"scenario {sc.name!r} has no host state")
        return cls(sc.grid, sc.params, sc.q0, sc.boundary, cfl=cfl, device=device, debug=debug,
                   rows_per_block=rows_per_block)

    def _init_on_device(self, ic):
        """The column-equilibrium initial condition built by the device
        (wb_init_column_equilibrium, bit-identical to ic.host_state)."""
        boxes = np.ascontiguousarray(np.array(ic.boxes, dtype=np.float64).reshape(-1))
        gas = math.nan if ic.gas_rho is None else float(ic.gas_rho)
        check(self._L.wb_init_column_equilibrium(
            self._h, len(ic.boxes), dptr(boxes) if len(ic.boxes) else None,
            float(ic.alpha_liq), float(ic.alpha_gas), gas), "wb_init_column_equilibrium")
        self._qh = None
        self._qh_exposed = False
        # host copies of the (unchanging) solid cells, for sim.q downloads
        self._solid_q = None
        if self._solid_flat.size:
            self._solid_q = self._get_q(0).reshape(-1, 5)[self._solid_flat].copy()

    def _host_q(self):
        """The current state on the host (cached until the next step)."""
        if self._qh is None:
            self._qh = self._get_q(0)
        return self._qh

    def _flush_q(self):
        """Upload a mirror the caller may have written through ``sim.q``
        (reference semantics: q is the live array)."""
        if self._qh is not None and self._qh_exposed:
            self._set_q(self._qh)

    def _stepped(self):
        self._qh = None
        self._qh_exposed = False

    @property
    def q(self):
        q = self._host_q()
        self._qh_exposed = True
        return q

    @q.setter
    def q(self, value):
        value = np.asarray(value, dtype=np.float64)
        if value.shape != (self.grid.nx, self.grid.ny, 5):
            raise SimulationError(f"q must have shape {(self.grid.nx, self.grid.ny, 5)}")
        self._set_q(value)

    def get_state(self, out=None):
        """Download the current state into ``out`` (an (nx, ny, 5) float64
        array, e.g. pinned host memory) or a new array; unlike ``sim.q`` it
        neither caches nor re-uploads."""
        self._flush_q()
        return self._get_q(0, out=out)

    @property
    def q_next(self):
        q = self._get_q(1)
        q.flags.writeable = False  # a copy: writes could not reach the device
        return q

    @property
    def t(self):
        return self._t

    @t.setter
    def t(self, value):
        self._t = float(value)
        check(self._L.wb_set_time(self._h, self._t, self._step), "wb_set_time")

    @property
    def step_count(self):
        return self._step

    @step_count.setter
    def step_count(self, value):
        self._step = int(value)
        check(self._L.wb_set_time(self._h, self._t, self._step), "wb_set_time")

    @property
    def edges(self):
        if self._edges is None:
            self._edges = EdgeSet(self.grid, self.boundary)
        return self._edges

    # ---- diagnostics --------------------------------------------------------
    @property
    def y0s(self):
        y0 = np.empty(self.grid.nx)
        check(self._L.wb_get_columns(self._h, dptr(y0), None), "wb_get_columns")
        return y0

    @property
    def aeqs(self):
        a = np.empty(self.grid.nx)
        check(self._L.wb_get_columns(self._h, None, dptr(a)), "wb_get_columns")
        return a

    def detect(self):
        """Column detection of the current state (timestepper.py:132-135)."""
        self._flush_q()
        r = ctypes.c_double()
        e = WbError()
        check(self._L.wb_max_rate(self._h, ctypes.byref(r), ctypes.byref(e)), "wb_max_rate")
        return self.y0s, self.aeqs

    def primitive_fields(self):
        """(rho, u, v, alpha, p); solid cells hold zeros (timestepper.py:107-125)."""
        q = self._host_q()
        fluid = self._fluid
        rho = np.zeros_like(q[:, :, 0])
        u = np.zeros_like(rho)
        v = np.zeros_like(rho)
        p = np.zeros_like(rho)
        alpha = np.where(fluid, q[:, :, 3], 0.0)
        np.divide(q[:, :, 0], q[:, :, 3], out=rho, where=fluid)
        np.divide(q[:, :, 1], q[:, :, 0], out=u, where=fluid)
        np.divide(q[:, :, 2], q[:, :, 0], out=v, where=fluid)
        pr = self.params
        if pr.gamma == 1.0:
            np.multiply(rho / pr.rho0 - 1.0, pr.k0, out=p, where=fluid)
        else:
            np.multiply((rho / pr.rho0) ** pr.gamma - 1.0, pr.k0, out=p, where=fluid)
        return rho, u, v, alpha, p

    def total_mass(self, device=False):
        """sum(alpha rho) * cell area over fluid cells (timestepper.py:127-130).

        The default downloads q and sums with numpy exactly like the
        reference; ``device=True`` uses the on-device deterministic reduction
        (no download; equal to ~1e-15 relative, different summation order)."""
        if device:
            return self.diagnostics()["mass"]
        return float(np.sum(self._host_q()[:, :, 0][self._fluid]) * self.grid.cell_area)

    def diagnostics(self, y0_eq=None):
        """Device-side reductions of the current state: mass, max |u|, max |v|,
        alpha range and -- given the surface level ``y0_eq`` of the exact
        water-at-rest profile -- the paper's equilibrium errors E_rho, E_u, E_v,
        E_P."""
        self._flush_q()
        out = np.empty(9)
        check(self._L.wb_diagnostics(self._h, math.nan if y0_eq is None else float(y0_eq),
                                     dptr(out)), "wb_diagnostics")
        keys = ("mass", "max_u", "max_v", "min_alpha", "max_alpha", "E_rho", "E_u", "E_v",
                "E_P")
        d = dict(zip(keys, (float(v) for v in out)))
        if y0_eq is None:
            for k in keys[5:]:
                d.pop(k)
        return d

    def depth_averaged_velocity(self):
        """u_bar(x) per column on the device (see analysis.depth_averaged_velocity
        for the host formula; same terms, j-ordered sums)."""
        self._flush_q()
        out = np.empty(self.grid.nx)
        check(self._L.wb_depth_averaged_velocity(self._h, dptr(out)),
              "wb_depth_averaged_velocity")
        return out

    # ---- errors -------------------------------------------------------------
    def _raise(self, e):
        if e.code == _lib.ERR_WAVE_SPEED:
            raise SimulationError(f"non-finite wave speed (max rate {float(e.rmax)})",
                                  step=int(e.step))
        q5 = np.empty(5)
        check(self._L.wb_get_cell(self._h, e.i, e.j, dptr(q5)), "wb_get_cell")
        raise SimulationError(f"{_MESSAGES[e.code]}; q = {q5}", step=int(e.step),
                              cell=(int(e.i), int(e.j)))

    def _sync_time(self):
        s = WbStatus()
        check(self._L.wb_get_status(self._h, ctypes.byref(s)), "wb_get_status")
        self._t = s.t
        self._step = int(s.step)
        return s

    def max_rate(self):
        """Detection + CFL rate max of the current state (timestepper.py:143-159)."""
        self._flush_q()
        r = ctypes.c_double()
        e = WbError()
        check(self._L.wb_max_rate(self._h, ctypes.byref(r), ctypes.byref(e)), "wb_max_rate")
        if e.code:
            self._raise(e)
        return r.value

    # ---- stepping -----------------------------------------------------------
    def advance(self, max_dt=None):
        """One step; returns the dt taken (timestepper.py:163-218)."""
        wall0 = time.perf_counter()
        self._flush_q()
        dt = ctypes.c_double()
        e = WbError()
        mdt = math.nan if max_dt is None else float(max_dt)
        if self.debug:
            arrs = WbStageArrays()
            for name in ("fW", "fE", "fS", "fN", "vol", "psi", "DW", "DE", "DS", "DN",
                         "rhoE_c", "rhoE_fy"):
                setattr(arrs, name, dptr(getattr(self, name)))
            arrs.quiet = u8ptr(self.quiet)
            check(self._L.wb_advance_debug(self._h, mdt, ctypes.byref(dt), ctypes.byref(e),
                                           ctypes.byref(arrs)), "wb_advance_debug")
        else:
            check(self._L.wb_advance(self._h, mdt, ctypes.byref(dt), ctypes.byref(e)),
                  "wb_advance")
        if e.code:
            self._raise(e)
        self._stepped()
        s = self._sync_time()
        wall = time.perf_counter() - wall0
        self.stats.dt = dt.value
        self.stats.max_rate = s.rmax
        self.stats.cells_per_second = self._n_fluid / wall if wall > 0.0 else 0.0
        return dt.value

    def run_until(self, t_end, callback=None, max_steps=None):
        """Advance to t_end, clamping the last step (timestepper.py:220-229).

        Without a callback the whole loop runs on the device (CUDA-graph
        chunks, one 8-byte status read per chunk); with a callback it steps
        from the host so the callback can observe every state."""
        if callback is not None or self.debug:
            tiny = 1.0e-12 * max(1.0, abs(t_end))
            while self._t < t_end - tiny:
                self.advance(max_dt=t_end - self._t)
                if callback is not None:
                    callback(self)
                if max_steps is not None and self._step >= max_steps:
                    break
            return self._t
        wall0 = time.perf_counter()
        step0 = self._step
        self._flush_q()
        e = WbError()
        check(self._L.wb_run(self._h, float(t_end), -1 if max_steps is None else int(max_steps),
                             16, ctypes.byref(e)), "wb_run")
        self._stepped()
        if e.code:
            self._sync_time()
            self._raise(e)
        s = self._sync_time()
        n = self._step - step0
        wall = time.perf_counter() - wall0
        if n:
            self.stats.dt = s.dt
            self.stats.max_rate = s.rmax
            self.stats.cells_per_second = self._n_fluid * n / wall if wall > 0 else 0.0
        return self._t

    def run_steps(self, n, chunk=16):
        """Device-side loop of exactly n steps (no time limit); n <= 0 takes
        no step (like DistributedSimulation.run_steps)."""
        if int(n) <= 0:
            return self._step
        self._flush_q()
        e = WbError()
        check(self._L.wb_run(self._h, math.nan, self._step + int(n), int(chunk),
                             ctypes.byref(e)), "wb_run")
        self._stepped()
        if e.code:
            self._sync_time()
            self._raise(e)
        self._sync_time()
        return self._step

    def eval_faces(self, kind, qm, qp, aux=None):
        """The device face solvers on arrays of state pairs with this
        simulation's physics (test hook, ``wb_eval_faces``): kind "x" =
        osher_x_edge, kind "y" = or_y_edge with aux rows (y, y0, aeq).  qm, qp
        are (n, 4); returns (D-, D+) as (n, 4) arrays."""
        qm = np.ascontiguousarray(qm, dtype=np.float64)
        qp = np.ascontiguousarray(qp, dtype=np.float64)
        n = qm.shape[0]
        if qm.shape != (n, 4) or qp.shape != (n, 4):
            raise ValueError("qm and qp must have shape (n, 4)")
        k = {"x": 0, "y": 1}[kind]
        ax = None
        if k == 1:
            ax = np.ascontiguousarray(aux, dtype=np.float64)
            if ax.shape != (n, 3):
                raise ValueError("aux must have shape (n, 3): (y, y0, aeq)")
        dm, dp = np.empty((n, 4)), np.empty((n, 4))
        check(self._L.wb_eval_faces(self._h, k, n, dptr(qm), dptr(qp),
                                    dptr(ax) if ax is not None else None, dptr(dm), dptr(dp)),
              "wb_eval_faces")
        return dm, dp

    def dt_log(self, n=None):
        n = self._step if n is None else n
        out = np.empty(n)
        check(self._L.wb_get_dt_log(self._h, dptr(out), n), "wb_get_dt_log")
        return out

    def work_counters(self):
        s = self._sync_time()
        return {"n_second_order": int(s.n_second_order), "x_faces": int(s.x_faces_solved),
                "y_faces": int(s.y_faces_solved), "n_fluid": self._n_fluid,
                "replays": int(s.replays),
                "replays_by_kind": dict(zip(("reconstruct", "flux_y_S", "x_face", "flux_x_pair",
                                             "y_face", "update"),
                                            (int(v) for v in s.replays_by_kind)))}


def compute_dt(sim, cfl=None):
    """cfl / max rate (timestepper.py:232-237)."""
    c = sim.cfl if cfl is None else float(cfl)
    if not 0.0 < c < 1.0:
        raise SimulationError(f"cfl must lie in (0, 1), got {c}")
    return c / sim.max_rate()


def advance_step(sim, max_dt=None):
    return sim.advance(max_dt=max_dt)


def total_mass(sim):
    return sim.total_mass()

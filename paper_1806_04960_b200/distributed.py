"""x-slab multi-GPU driver.

One process per GPU; rank r owns the global columns [i0, i1) of the grid plus
a 2-column halo on each side (update(i) needs q(i +- 2); detection is a
per-column reduction over j, so it stays local and bit-identical).  Per step,
all stream-ordered on the slab's CUDA stream (no host synchronisation):

    wb_step_local     detect + fused step kernel + [enc(errkey), rate] vector
    all_reduce(MAX)   -> globally first failing cell and the global CFL rate
    wb_finalize       commit (or stop) identically on every rank
    halo exchange     the edge columns stored into the neighbours' halo over
                      peer memory (before the all-reduce), or pack, send/recv
                      to the x-neighbours, unpack

Results are bit-identical to a single-GPU run (tests/test_distributed_cpu.py
runs the same driver over gloo with the CPU oracle as the slab backend).
``torch.distributed`` is the plumbing (NCCL on GPUs, gloo in the CPU tests);
the slab backends implement the same small interface:

    red, send, recv                tensors the collectives operate on
    prepare_local/pack/unpack()    first-step admissibility + rate
    check_prepare()                -> (rmax, code, key) after the reduction
    step_local(max_dt, t_end, mode), finalize(), pack_halo(), unpack_halo(l, r)
    status() -> dict, cell_q(i, j), owned_state()
"""

import contextlib
import ctypes
import math
import os

import numpy as np

from .errors import SimulationError

__all__ = ["slab_bounds", "stored_range", "DeviceSlab", "DistributedSimulation"]

HALO = 2
ENC_TOP = 1 << 62
_MESSAGES = {1: "non-admissible cell state",
             3: "non-admissible reconstructed face state",
             4: "negative mass or volume fraction after update"}


def slab_bounds(nx, world, rank):
    """Contiguous column range of `rank` (the first nx % world ranks get one
    extra column)."""
    base, extra = divmod(nx, world)
    i0 = rank * base + min(rank, extra)
    return i0, i0 + base + (1 if rank < extra else 0)


def stored_range(nx, i0, i1):
    """Columns a slab holds: owned plus the in-domain halo."""
    return max(0, i0 - HALO), min(nx, i1 + HALO)


def dec_key(e):
    return None if e == 0 else ENC_TOP - e


class _CudaArray:
    """__cuda_array_interface__ view of device memory owned by the library,
    so torch collectives can operate on it in place."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


class DeviceSlab:
    """Slab backend on one GPU through the C ABI (include/wbflow_b200.h)."""

    def __init__(self, grid, params, q_cols, col0, boundary, cfl, i0, i1, device, ic=None):
        """q_cols: the state of the stored columns [col0, col0 + n) (host); or
        None with ``ic`` (a scenarios.ColumnEquilibriumIC) to build this
        slab's columns on the device (wb_init_column_equilibrium)."""
        import torch
        from . import _lib
        from .timestepper import make_config
        self.torch = torch
        self._lib = _lib
        self.L = _lib.load()
        self.grid = grid
        self.i0, self.i1, self.ny = i0, i1, grid.ny
        torch.cuda.set_device(device)
        cfg = make_config(grid, params, boundary, cfl, i_begin=i0, i_end=i1, device=device)
        mask = np.ascontiguousarray(grid.mask, dtype=np.uint8)
        xc = np.ascontiguousarray(grid.x_centers)
        yc = np.ascontiguousarray(grid.y_centers)
        yf = np.ascontiguousarray(grid.y_faces)
        h = ctypes.c_void_p()
        _lib.check(self.L.wb_create(ctypes.byref(cfg), _lib.u8ptr(mask), _lib.dptr(xc),
                                    _lib.dptr(yc), _lib.dptr(yf), ctypes.byref(h)), "wb_create")
        self.h = h
        self.stream = torch.cuda.Stream(device=device)
        _lib.check(self.L.wb_set_stream(h, ctypes.c_void_p(self.stream.cuda_stream)),
                   "wb_set_stream")
        # slab-edge strips + halo exchange (overlapped step); high priority so
        # the boundary columns are done early and the exchange starts early
        self.edge_stream = torch.cuda.Stream(device=device, priority=-1)
        _lib.check(self.L.wb_set_edge_stream(h, ctypes.c_void_p(self.edge_stream.cuda_stream)),
                   "wb_set_edge_stream")
        if q_cols is None:
            boxes = np.ascontiguousarray(np.array(ic.boxes, dtype=np.float64).reshape(-1))
            _lib.check(self.L.wb_init_column_equilibrium(
                h, len(ic.boxes), _lib.dptr(boxes) if len(ic.boxes) else None,
                float(ic.alpha_liq), float(ic.alpha_gas),
                math.nan if ic.gas_rho is None else float(ic.gas_rho)),
                "wb_init_column_equilibrium")
        else:
            q = np.ascontiguousarray(q_cols, dtype=np.float64)
            bi, bj = ctypes.c_int32(), ctypes.c_int32()
            _lib.check(self.L.wb_set_state(h, q.ctypes.data_as(ctypes.c_void_p), col0,
                                           q.shape[0], 0, ctypes.byref(bi), ctypes.byref(bj)),
                       "wb_set_state")
        rp = ctypes.c_void_p()
        _lib.check(self.L.wb_reduce_ptr(h, ctypes.byref(rp)), "wb_reduce_ptr")
        self.red = torch.as_tensor(_CudaArray(rp.value, 2, "<i8"), device=f"cuda:{device}")
        n = ctypes.c_int64()
        _lib.check(self.L.wb_halo_count(h, ctypes.byref(n)), "wb_halo_count")
        self.send = torch.zeros(n.value, dtype=torch.float64, device=f"cuda:{device}")
        self.recv = torch.zeros(n.value, dtype=torch.float64, device=f"cuda:{device}")
        self._n_fluid = None  # counted on first use (not part of an upload)

    @property
    def n_fluid(self):
        if self._n_fluid is None:
            self._n_fluid = int(np.count_nonzero(np.asarray(self.grid.mask)[self.i0:self.i1]))
        return self._n_fluid

    def stream_ctx(self):
        return self.torch.cuda.stream(self.stream)

    def edge_ctx(self):
        return self.torch.cuda.stream(self.edge_stream)

    def step_begin(self, max_dt, t_end, mode):
        self._lib.check(self.L.wb_step_begin(self.h, math.nan if max_dt is None else max_dt,
                                             0.0 if t_end is None else t_end, mode,
                                             ctypes.c_void_p(self.send.data_ptr())),
                        "wb_step_begin")

    # -- halo over peer memory (wb_set_peers) --
    def peer_desc(self):
        """This slab's buffers (wb_peer) for a neighbour in the same process."""
        p = self._lib.WbPeer()
        self._lib.check(self.L.wb_peer_desc(self.h, ctypes.byref(p)), "wb_peer_desc")
        return p

    def peer_export(self):
        """This slab's buffers as a CUDA IPC blob for another process."""
        b = ctypes.create_string_buffer(self._lib.WB_PEER_IPC_BYTES)
        self._lib.check(self.L.wb_peer_ipc_export(self.h, b), "wb_peer_ipc_export")
        return bytes(b.raw)

    def peer_open(self, blob):
        """A neighbour's exported buffers, opened on this slab's device."""
        p = self._lib.WbPeer()
        b = ctypes.create_string_buffer(bytes(blob), self._lib.WB_PEER_IPC_BYTES)
        self._lib.check(self.L.wb_peer_ipc_open(self.h, b, ctypes.byref(p)), "wb_peer_ipc_open")
        return p

    def set_peers(self, left, right):
        self._lib.check(self.L.wb_set_peers(self.h, ctypes.byref(left) if left else None,
                                            ctypes.byref(right) if right else None),
                        "wb_set_peers")
        self.peers = (left, right)  # keep the descriptors alive

    def step_begin_peer(self, max_dt, t_end, mode):
        self._lib.check(self.L.wb_step_begin_peer(self.h, math.nan if max_dt is None else max_dt,
                                                  0.0 if t_end is None else t_end, mode),
                        "wb_step_begin_peer")

    def push_halo_next(self):
        self._lib.check(self.L.wb_push_halo_next(self.h), "wb_push_halo_next")

    def unpack_halo_next(self, have_left, have_right):
        self._lib.check(self.L.wb_unpack_halo_next(self.h, ctypes.c_void_p(self.recv.data_ptr()),
                                                   int(have_left), int(have_right)),
                        "wb_unpack_halo_next")

    def step_end(self):
        self._lib.check(self.L.wb_step_end(self.h), "wb_step_end")

    def prepare_local(self):
        self._lib.check(self.L.wb_prepare_local(self.h), "wb_prepare_local")

    def prepare_pack(self):
        self._lib.check(self.L.wb_prepare_pack(self.h), "wb_prepare_pack")

    def prepare_unpack(self):
        self._lib.check(self.L.wb_prepare_unpack(self.h), "wb_prepare_unpack")

    def check_prepare(self):
        from ._lib import WbError
        r, e = ctypes.c_double(), WbError()
        self._lib.check(self.L.wb_check_prepare(self.h, ctypes.byref(r), ctypes.byref(e)),
                        "wb_check_prepare")
        key = None if e.i < 0 else e.i * self.ny + e.j
        return r.value, e.code, key

    def step_local(self, max_dt, t_end, mode):
        self._lib.check(self.L.wb_step_local(self.h, math.nan if max_dt is None else max_dt,
                                             0.0 if t_end is None else t_end, mode),
                        "wb_step_local")

    def finalize(self):
        self._lib.check(self.L.wb_finalize(self.h), "wb_finalize")

    def pack_halo(self):
        self._lib.check(self.L.wb_pack_halo(self.h, ctypes.c_void_p(self.send.data_ptr())),
                        "wb_pack_halo")

    def unpack_halo(self, have_left, have_right):
        self._lib.check(self.L.wb_unpack_halo(self.h, ctypes.c_void_p(self.recv.data_ptr()),
                                              int(have_left), int(have_right)), "wb_unpack_halo")

    def status(self):
        from ._lib import WbStatus
        s = WbStatus()
        self._lib.check(self.L.wb_get_status(self.h, ctypes.byref(s)), "wb_get_status")
        return {"t": s.t, "dt": s.dt, "step": int(s.step), "stop": int(s.stop),
                "rmax": s.rmax, "counters": (int(s.n_second_order), int(s.x_faces_solved),
                                             int(s.y_faces_solved))}

    def last_error(self):
        """(code, global key or None, step, rmax) recorded by the finalize
        kernel when the run stopped on an error."""
        from ._lib import WbError
        e = WbError()
        self._lib.check(self.L.wb_get_error(self.h, ctypes.byref(e)), "wb_get_error")
        key = None if e.i < 0 else e.i * self.ny + e.j
        return e.code, key, int(e.step), e.rmax

    def cell_q(self, i, j):
        q5 = np.empty(5)
        self._lib.check(self.L.wb_get_cell(self.h, i, j, self._lib.dptr(q5)), "wb_get_cell")
        return q5

    def owned_state(self):
        q = np.empty((self.i1 - self.i0, self.ny, 5))
        self._lib.check(self.L.wb_get_state(self.h, q.ctypes.data_as(ctypes.c_void_p), 0),
                        "wb_get_state")
        return q


class DistributedSimulation:
    """x-slab decomposition of one simulation over the ranks of a
    torch.distributed process group (the reference's Simulation semantics:
    same dt sequence, same error step/cell, bit-identical state)."""

    def __init__(self, backend, grid, cfl=0.45, group=None, overlap=True, graphs=True,
                 halo=None):
        import torch.distributed as dist
        self.dist = dist
        self.be = backend
        self.grid = grid
        self.cfl = cfl
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.t = 0.0
        self.step_count = 0
        self._prepared = False
        self._nccl = dist.get_backend(group) == "nccl"
        # overlapped step (default): edge strips + halo exchange on the
        # backend's edge stream while the interior strips run (SURVEY.md 8(e)
        # "Overlap").  The edge strips detect their columns with a one-warp-
        # per-column kernel instead of the fused chain, so on one B200 the
        # split step costs the same as the plain one (6.654 vs 6.658 ms on the
        # C5 slab, tools/overlap_bench.py) and hides the exchange on several.
        self.overlap = overlap and hasattr(backend, "step_begin")
        # device loops over NCCL are captured once per chunk length as a CUDA
        # graph (kernels + collectives), replayed without host enqueue work;
        # set to False after a failed capture (then steps are enqueued eagerly)
        self.use_graphs = graphs and self._nccl and hasattr(backend, "stream")
        self._graphs = {}
        # halo exchange: "peer" -- the step kernel's boundary columns stored by
        # one kernel straight into the neighbours' halo (NVLink stores between
        # GPUs, CUDA IPC between processes; the default for device slabs), or
        # "collective" -- pack, send/recv through torch.distributed, unpack
        if halo is None:
            halo = os.environ.get("WB_HALO", "peer" if hasattr(backend, "peer_export")
                                  else "collective")
        if halo not in ("peer", "collective"):
            raise ValueError(f"halo must be 'peer' or 'collective', not {halo!r}")
        self.halo = halo
        if halo == "peer":
            self._setup_peers()

    def _setup_peers(self):
        """Every rank exports its buffers (CUDA IPC), gathers the others' and
        opens its x-neighbours' on its device; falls back to the collective
        exchange (with a warning) where peer access is unavailable."""
        be, r, W = self.be, self.rank, self.world
        try:
            blobs = [None] * W
            self.dist.all_gather_object(blobs, be.peer_export(), group=self.group)
            left = be.peer_open(blobs[r - 1]) if r > 0 else None
            right = be.peer_open(blobs[r + 1]) if r < W - 1 else None
            be.set_peers(left, right)
            ok = 1
        except Exception as e:  # noqa: BLE001 -- reported, then the other path
            import warnings
            warnings.warn(f"halo over peer memory unavailable ({e}); using send/recv")
            ok = 0
        # every rank must take the same path
        import torch
        t = torch.tensor([ok], dtype=torch.int64,
                         device=be.red.device if self._nccl else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        if int(t.item()) == 0:
            if ok:
                be.set_peers(None, None)
            self.halo = "collective"

    # -- collectives ------------------------------------------------------
    def _allreduce_max(self, t):
        if t.is_cuda and not self._nccl:  # gloo with device slabs: stage through host
            h = t.cpu()
            self.dist.all_reduce(h, op=self.dist.ReduceOp.MAX, group=self.group)
            t.copy_(h)
            return
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)

    def _halo_exchange(self):
        self.be.pack_halo()
        self._p2p()
        self.be.unpack_halo(self.rank > 0, self.rank < self.world - 1)

    def _p2p(self):
        """send/recv of the packed halo blocks with the x-neighbours on the
        current stream (NCCL), or through host copies (gloo)."""
        be, r, W = self.be, self.rank, self.world
        half = be.send.numel() // 2
        staged = be.send.is_cuda and not self._nccl  # gloo: point-to-point on host copies
        send, recv = (be.send.cpu(), be.recv.cpu()) if staged else (be.send, be.recv)
        ops = []
        P2P = self.dist.P2POp
        if r > 0:
            ops.append(P2P(self.dist.isend, send[:half], r - 1, self.group))
            ops.append(P2P(self.dist.irecv, recv[:half], r - 1, self.group))
        if r < W - 1:
            ops.append(P2P(self.dist.isend, send[half:], r + 1, self.group))
            ops.append(P2P(self.dist.irecv, recv[half:], r + 1, self.group))
        if ops:
            if self._nccl:
                for w in self.dist.batch_isend_irecv(ops):
                    w.wait()
            else:
                reqs = [op.op(op.tensor, op.peer, op.group) for op in ops]
                for q in reqs:
                    q.wait()
        if staged:
            be.recv.copy_(recv)

    def _ctx(self):
        return self.be.stream_ctx() if hasattr(self.be, "stream_ctx") else \
            contextlib.nullcontext()

    # -- prepare (first step after an upload) ---------------------------------
    def prepare(self):
        be = self.be
        with self._ctx():
            be.prepare_local()
            be.prepare_pack()
            self._allreduce_max(be.red)
            be.prepare_unpack()
        rmax, code, key = be.check_prepare()
        if code == 1:
            i, j = divmod(key, self.grid.ny)
            raise SimulationError(f"{_MESSAGES[1]}; q = {self._cell_q(i, j)}",
                                  step=self.step_count, cell=(i, j))
        if code == 2:
            raise SimulationError(f"non-finite wave speed (max rate {rmax})",
                                  step=self.step_count)
        self._prepared = True
        return rmax

    # -- stepping -----------------------------------------------------------
    def _edge_ctx(self):
        return self.be.edge_ctx() if hasattr(self.be, "edge_ctx") else contextlib.nullcontext()

    def _enqueue_step(self, max_dt=None, t_end=None):
        be = self.be
        mode = 1 if t_end is not None else 0
        if self.halo == "peer":
            # the halo goes into the neighbours' step output buffers before the
            # all-reduce, which orders it before any rank's next step
            with self._ctx():
                if self.overlap:
                    be.step_begin_peer(max_dt, t_end, mode)  # edges + peer stores on edge
                    be.step_end()
                else:
                    be.step_local(max_dt, t_end, mode)
                    be.push_halo_next()
                self._allreduce_max(be.red)
                be.finalize()
            return
        if self.overlap:
            with self._ctx():
                be.step_begin(max_dt, t_end, mode)  # interior here, edges + pack on edge
            with self._edge_ctx():
                self._p2p()
                be.unpack_halo_next(self.rank > 0, self.rank < self.world - 1)
            with self._ctx():
                be.step_end()                       # join the edge stream
                self._allreduce_max(be.red)
                be.finalize()
            return
        with self._ctx():
            be.step_local(max_dt, t_end, 1 if t_end is not None else 0)
            self._allreduce_max(be.red)
            be.finalize()
            self._halo_exchange()

    def enqueue_steps(self, n):
        """Enqueue n steps (mode 0: no time limit) without a host sync: as
        replays of a captured CUDA graph of the step sequence (step kernels,
        MAX all-reduce, finalize, halo send/recv) when the group is NCCL, else
        eagerly."""
        if not self._prepared:
            self.prepare()
        if not self.use_graphs:
            for _ in range(n):
                self._enqueue_step()
            return
        torch = self.be.torch
        g = self._graphs.get(n)
        if g is None:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g, stream=self.be.stream):
                    for _ in range(n):
                        self._enqueue_step()
            except Exception as e:  # capture unsupported here: eager from now on
                import warnings
                warnings.warn(f"CUDA graph capture of the distributed step failed ({e}); "
                              "enqueueing steps eagerly")
                self.use_graphs = False
                torch.cuda.synchronize()
                for _ in range(n):
                    self._enqueue_step()
                return
            self._graphs[n] = g
        with self._ctx():  # a graph replays on the current stream: the backend's
            g.replay()

    def _sync(self):
        s = self.be.status()
        self.t, self.step_count = s["t"], s["step"]
        return s

    def _cell_q(self, i, j):
        """q of global cell (i, j) from its owner, via a SUM all-reduce."""
        import torch
        owner = self.be.i0 <= i < self.be.i1
        # non-owners contribute -0.0, the exact identity of IEEE addition
        # (+0.0 would turn a -0.0 component of the owner's cell into +0.0)
        q = self.be.cell_q(i, j) if owner else np.full(5, -0.0)
        dev = self.be.red.device
        with self._ctx():  # the H2D copy and the collective on the same stream
            t = torch.tensor(q, dtype=torch.float64, device=dev if self._nccl else "cpu")
            self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def _check(self, s):
        if s["stop"] > 0:
            code, key, step, rmax = self.be.last_error()
            if code == 2:
                raise SimulationError(f"non-finite wave speed (max rate {rmax})", step=step)
            i, j = divmod(key, self.grid.ny)
            raise SimulationError(f"{_MESSAGES[code]}; q = {self._cell_q(i, j)}", step=step,
                                  cell=(i, j))

    def advance(self, max_dt=None):
        if not self._prepared:
            self.prepare()
        self._enqueue_step(max_dt=max_dt)
        s = self._sync()
        self._check(s)
        return s["dt"]

    def run_steps(self, n, check_every=16):
        if not self._prepared:
            self.prepare()
        done = 0
        while done < n:
            k = min(check_every, n - done)
            self.enqueue_steps(k)
            done += k
            s = self._sync()
            self._check(s)
        return self.step_count

    def run_until(self, t_end, max_steps=None):
        if not self._prepared:
            self.prepare()
        tiny = 1.0e-12 * max(1.0, abs(t_end))
        while self.t < t_end - tiny:
            self._enqueue_step(t_end=t_end)
            s = self._sync()
            self._check(s)
            if max_steps is not None and self.step_count >= max_steps:
                break
        return self.t

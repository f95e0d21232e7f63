"""ctypes binding of libwbflow_b200.so (include/wbflow_b200.h).

This is the only way the package reaches the device.  There is no CPU
fallback: if the library is missing or no CUDA device is present, every
entry point raises ``DeviceError``.
"""

import ctypes
import os

from .errors import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
# WB_LIB_PATH: load another build of the same sources (measurement experiments
# such as tools/exp_nocheck.sh); the default is the in-tree library
LIB_PATH = os.environ.get("WB_LIB_PATH") or os.path.join(_HERE, "libwbflow_b200.so")

WB_OK = 0
WB_E_ARG, WB_E_CUDA, WB_E_HEIGHT, WB_E_STATE = -1, -2, -3, -4
ERR_CELL_STATE, ERR_WAVE_SPEED, ERR_FACE, ERR_MASS = 1, 2, 3, 4

c_double_p = ctypes.POINTER(ctypes.c_double)
c_u8_p = ctypes.POINTER(ctypes.c_uint8)


class WbConfig(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("i_begin", ctypes.c_int32), ("i_end", ctypes.c_int32),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double),
                ("k0", ctypes.c_double), ("rho0", ctypes.c_double),
                ("gamma", ctypes.c_double), ("g", ctypes.c_double),
                ("epsilon", ctypes.c_double), ("cfl", ctypes.c_double),
                ("bc_kind", ctypes.c_int32 * 4),
                ("inflow_seg", (ctypes.c_double * 2) * 4),
                ("inflow_q", (ctypes.c_double * 4) * 4),
                ("device", ctypes.c_int32), ("rows_per_block", ctypes.c_int32)]


class WbError(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("step", ctypes.c_int64),
                ("i", ctypes.c_int32), ("j", ctypes.c_int32), ("rmax", ctypes.c_double)]


class WbStatus(ctypes.Structure):
    _fields_ = [("t", ctypes.c_double), ("dt", ctypes.c_double), ("rmax", ctypes.c_double),
                ("step", ctypes.c_int64), ("stop", ctypes.c_int32), ("cur", ctypes.c_int32),
                ("n_second_order", ctypes.c_uint64), ("x_faces_solved", ctypes.c_uint64),
                ("y_faces_solved", ctypes.c_uint64), ("replays", ctypes.c_uint64),
                ("replays_by_kind", ctypes.c_uint64 * 6)]


class WbPeer(ctypes.Structure):
    """wb_peer: an x-neighbour slab's buffers as pointers on this device."""
    _fields_ = [("q", (ctypes.c_void_p * 4) * 2), ("y0s", ctypes.c_void_p * 2),
                ("aeqs", ctypes.c_void_p * 2), ("pitch", ctypes.c_int32),
                ("nxl", ctypes.c_int32), ("ny", ctypes.c_int32), ("pad", ctypes.c_int32)]


WB_PEER_IPC_BYTES = 256


class WbStageArrays(ctypes.Structure):
    _fields_ = [(n, c_double_p) for n in ("fW", "fE", "fS", "fN", "vol", "psi", "DW", "DE",
                                          "DS", "DN", "rhoE_c", "rhoE_fy")] + \
               [("quiet", c_u8_p)]


# name -> (restype, argtypes); every function returns int status
_H = ctypes.c_void_p
_V = ctypes.c_void_p
SIGNATURES = {
    "wb_create": [ctypes.POINTER(WbConfig), c_u8_p, c_double_p, c_double_p, c_double_p,
                  ctypes.POINTER(_H)],
    "wb_destroy": [_H],
    "wb_set_stream": [_H, _V],
    "wb_set_state": [_H, _V, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                     ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)],
    "wb_get_state": [_H, _V, ctypes.c_int32],
    "wb_init_column_equilibrium": [_H, ctypes.c_int32, c_double_p, ctypes.c_double,
                                   ctypes.c_double, ctypes.c_double],
    "wb_get_state_buf": [_H, _V, ctypes.c_int32, ctypes.c_int32],
    "wb_get_cell": [_H, ctypes.c_int32, ctypes.c_int32, c_double_p],
    "wb_max_rate": [_H, c_double_p, ctypes.POINTER(WbError)],
    "wb_get_columns": [_H, c_double_p, c_double_p],
    "wb_advance": [_H, ctypes.c_double, c_double_p, ctypes.POINTER(WbError)],
    "wb_run": [_H, ctypes.c_double, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(WbError)],
    "wb_get_status": [_H, ctypes.POINTER(WbStatus)],
    "wb_get_error": [_H, ctypes.POINTER(WbError)],
    "wb_diagnostics": [_H, ctypes.c_double, c_double_p],
    "wb_set_time": [_H, ctypes.c_double, ctypes.c_int64],
    "wb_get_dt_log": [_H, c_double_p, ctypes.c_int64],
    "wb_advance_debug": [_H, ctypes.c_double, c_double_p, ctypes.POINTER(WbError),
                         ctypes.POINTER(WbStageArrays)],
    "wb_reduce_ptr": [_H, ctypes.POINTER(_V)],
    "wb_prepare_ptrs": [_H, ctypes.POINTER(_V), ctypes.POINTER(_V)],
    "wb_prepare_local": [_H],
    "wb_prepare_pack": [_H],
    "wb_prepare_unpack": [_H],
    "wb_get_stream": [_H, ctypes.POINTER(_V)],
    "wb_check_prepare": [_H, c_double_p, ctypes.POINTER(WbError)],
    "wb_step_local": [_H, ctypes.c_double, ctypes.c_double, ctypes.c_int32],
    "wb_finalize": [_H],
    "wb_halo_count": [_H, ctypes.POINTER(ctypes.c_int64)],
    "wb_pack_halo": [_H, _V],
    "wb_unpack_halo": [_H, _V, ctypes.c_int32, ctypes.c_int32],
    "wb_set_edge_stream": [_H, _V],
    "wb_step_begin": [_H, ctypes.c_double, ctypes.c_double, ctypes.c_int32, _V],
    "wb_unpack_halo_next": [_H, _V, ctypes.c_int32, ctypes.c_int32],
    "wb_step_end": [_H],
    "wb_peer_desc": [_H, ctypes.POINTER(WbPeer)],
    "wb_peer_ipc_export": [_H, _V],
    "wb_peer_ipc_open": [_H, _V, ctypes.POINTER(WbPeer)],
    "wb_set_peers": [_H, ctypes.POINTER(WbPeer), ctypes.POINTER(WbPeer)],
    "wb_step_begin_peer": [_H, ctypes.c_double, ctypes.c_double, ctypes.c_int32],
    "wb_push_halo_next": [_H],
    "wb_eval_faces": [_H, ctypes.c_int32, ctypes.c_int64, _V, _V, _V, _V, _V],
    "wb_depth_averaged_velocity": [_H, _V],
    "wb_sync": [_H],
    "wb_profile_steps": [_H, ctypes.c_int32, c_double_p, c_double_p, c_double_p],
    "wb_fp64_peak": [ctypes.c_int32, c_double_p],
    "wb_eval_exp": [ctypes.c_int32, c_double_p, c_double_p, ctypes.c_int64],
    "wb_selftest_div": [ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                        ctypes.POINTER(ctypes.c_uint64)],
    "wb_version": [],
}

_lib = None


def load(build_if_missing=True):
    """Load (building in-tree first if needed) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing:
        from .build import build
        build()
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as e:
        raise DeviceError(f"cannot load {LIB_PATH}: {e}") from e
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = ctypes.c_int
        fn.argtypes = args
    lib.wb_last_error.restype = ctypes.c_char_p
    lib.wb_last_error.argtypes = []
    _lib = lib
    return lib


def check(rc, what=""):
    if rc != WB_OK:
        msg = load().wb_last_error().decode(errors="replace")
        raise DeviceError(f"{what} failed (status {rc}): {msg}")
    return rc


def dptr(a):
    return a.ctypes.data_as(c_double_p)


def u8ptr(a):
    return a.ctypes.data_as(c_u8_p)

"""Thin ctypes binding of include/chemora.h (argument marshalling only).

Every function here has the name of the C entry point it calls and does nothing but
convert arguments and raise ``ChemoraError`` on a non-OK status.  All arithmetic of the
method runs in the CUDA kernels of ``libchemora.so``; there is no CPU fallback: if the
library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libchemora.so")

SYS_WAVE, SYS_BSSN = 1, 2
N_GF = {SYS_WAVE: 5, SYS_BSSN: 25}
INIT_HOST, INIT_HOST_PADDED, INIT_PLANE_WAVES, INIT_GAUSSIAN, INIT_NOISE, INIT_MINK_PERT, INIT_GAUGE_WAVE = range(7)
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_SHAPE", 3: "E_NOMEM", 4: "E_CUDA", 5: "E_PEER",
          6: "E_NONFINITE", 7: "E_UNSUPPORTED"}
E_NONFINITE = 6

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1410_1764_b200.build` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)


class ChemoraError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = _lib.chemora_last_error().decode()
        super().__init__(f"{where}: {STATUS.get(code, code)}: {msg}")
        self.code = code


class chemora_grid_desc(ctypes.Structure):
    _fields_ = [("system", ctypes.c_int32), ("ghost", ctypes.c_int32), ("n_gf", ctypes.c_int32),
                ("device", ctypes.c_int32), ("extent", ctypes.c_int64 * 3),
                ("origin", ctypes.c_double * 3), ("spacing", ctypes.c_double * 3),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("fd_order", ctypes.c_int32),
                ("n_params", ctypes.c_int32), ("params", ctypes.POINTER(ctypes.c_double))]


_vp, _dp, _i64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
_descp = ctypes.POINTER(chemora_grid_desc)
_SIGS = {
    "chemora_version": ([], ctypes.c_char_p),
    "chemora_last_error": ([], ctypes.c_char_p),
    "chemora_grid_required_bytes": ([_descp, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "chemora_grid_create": ([_descp, _vp, ctypes.c_size_t, ctypes.POINTER(_vp)], ctypes.c_int),
    "chemora_grid_destroy": ([_vp], ctypes.c_int),
    "chemora_grid_local": ([_vp, _i64p, _i64p], ctypes.c_int),
    "chemora_set_initial": ([_vp, ctypes.c_int, _dp, _dp, ctypes.c_uint64, _vp], ctypes.c_int),
    "chemora_set_initial_nofill": ([_vp, ctypes.c_int, _dp, _dp, ctypes.c_uint64, _vp], ctypes.c_int),
    "chemora_get_state": ([_vp, _dp, _vp], ctypes.c_int),
    "chemora_get_state_padded": ([_vp, _dp, _vp], ctypes.c_int),
    "chemora_upload_state": ([_vp, _vp, _vp], ctypes.c_int),
    "chemora_download_state": ([_vp, _vp, _vp], ctypes.c_int),
    "chemora_rhs": ([_vp, _vp, _vp], ctypes.c_int),
    "chemora_rk4_step": ([_vp, ctypes.c_double, ctypes.c_int32, _vp], ctypes.c_int),
    "chemora_rk4_step_multi": ([ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_double,
                                ctypes.c_int32, _vp], ctypes.c_int),
    "chemora_halo_exchange": ([_vp, _vp], ctypes.c_int),
    "chemora_halo_exchange_multi": ([ctypes.POINTER(_vp), ctypes.c_int32, _vp], ctypes.c_int),
    "chemora_norms_partial": ([_vp, _dp, _vp], ctypes.c_int),
    "chemora_norms_combine": ([_descp, _dp, ctypes.c_int32, _dp], ctypes.c_int),
    "chemora_norms_len": ([ctypes.c_int32, ctypes.c_int32], ctypes.c_int),
    "chemora_norms": ([_vp, _dp, _vp], ctypes.c_int),
    "chemora_constraints": ([_vp, _vp, _dp, _vp], ctypes.c_int),
    "chemora_constraint_norms": ([_vp, _dp, _vp], ctypes.c_int),
    "chemora_grid_connect_local": ([ctypes.POINTER(_vp), ctypes.c_int32], ctypes.c_int),
    "chemora_peer_record_size": ([ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "chemora_grid_export_peer": ([_vp, _vp], ctypes.c_int),
    "chemora_grid_connect_ipc": ([_vp, _vp, _vp], ctypes.c_int),
    "chemora_set_kernel_variant": ([_vp, ctypes.c_int], ctypes.c_int),
    "chemora_set_monitor": ([_vp, ctypes.c_int], ctypes.c_int),
    "chemora_debug_get_set": ([_vp, ctypes.c_int, _dp, _vp], ctypes.c_int),
    "chemora_get_kernel_variant": ([_vp, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "chemora_read_monitor": ([_vp, _dp, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), _vp], ctypes.c_int),
    "chemora_autotune": ([_vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), _dp, _vp], ctypes.c_int),
    "chemora_read_monitor_multi": ([ctypes.POINTER(_vp), ctypes.c_int32, _dp, ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_int32), _vp], ctypes.c_int),
    "chemora_set_phase_barrier": ([_vp, _vp, _vp], ctypes.c_int),
    "chemora_set_launch_timing": ([_vp, ctypes.c_int], ctypes.c_int),
    "chemora_read_launch_timing": ([_vp, _dp, ctypes.POINTER(ctypes.c_int32), _vp], ctypes.c_int),
    "chemora_constraint_norms_combine": ([_descp, _dp, ctypes.c_int32, _dp], ctypes.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


def _check(rc: int, where: str):
    if rc != 0:
        raise ChemoraError(rc, where)


def _dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def make_desc(system, extent, spacing, origin=(0.0, 0.0, 0.0), ghost=3, device=0, rank=0,
              nranks=1, fd_order=0, params=None) -> chemora_grid_desc:
    d = chemora_grid_desc()
    d.system = system
    d.ghost = ghost
    d.n_gf = N_GF[system]
    d.device = device
    d.extent[:] = [int(v) for v in extent]
    d.origin[:] = [float(v) for v in origin]
    d.spacing[:] = [float(v) for v in spacing]
    d.rank, d.nranks, d.fd_order = rank, nranks, fd_order
    if params is not None:
        arr = (ctypes.c_double * len(params))(*[float(v) for v in params])
        d._params_keepalive = arr
        d.params = ctypes.cast(arr, _dp)
        d.n_params = len(params)
    else:
        d.params = None
        d.n_params = 0
    return d


# ------------------------------------------------------------------ raw entry points
def chemora_version() -> str:
    return _lib.chemora_version().decode()


def chemora_last_error() -> str:
    return _lib.chemora_last_error().decode()


def chemora_grid_required_bytes(desc) -> int:
    n = ctypes.c_size_t()
    _check(_lib.chemora_grid_required_bytes(ctypes.byref(desc), ctypes.byref(n)), "chemora_grid_required_bytes")
    return n.value


def chemora_grid_create(desc, workspace_ptr: int, nbytes: int):
    h = _vp()
    _check(_lib.chemora_grid_create(ctypes.byref(desc), _vp(workspace_ptr), nbytes, ctypes.byref(h)),
           "chemora_grid_create")
    return h


def chemora_grid_destroy(h):
    _check(_lib.chemora_grid_destroy(h), "chemora_grid_destroy")


def chemora_grid_local(h):
    ext = (ctypes.c_int64 * 3)()
    z0 = ctypes.c_int64()
    _check(_lib.chemora_grid_local(h, ext, ctypes.byref(z0)), "chemora_grid_local")
    return tuple(ext), z0.value


def chemora_set_initial(h, kind, host_src=None, kind_params=None, seed=0, stream=None, fill=True):
    kp = None if kind_params is None else np.ascontiguousarray(kind_params, dtype=np.float64)
    src = None if host_src is None else np.ascontiguousarray(host_src, dtype=np.float64)
    fn = _lib.chemora_set_initial if fill else _lib.chemora_set_initial_nofill
    _check(fn(h, kind, _dptr(src), _dptr(kp), seed, stream), "chemora_set_initial")


def chemora_get_state(h, out: np.ndarray, stream=None, padded=False, allow_nonfinite=False):
    fn = _lib.chemora_get_state_padded if padded else _lib.chemora_get_state
    rc = fn(h, _dptr(out), stream)
    if rc == E_NONFINITE and allow_nonfinite:
        return rc
    _check(rc, "chemora_get_state")
    return rc


def chemora_upload_state(h, host_ptr: int, stream=None):
    """Stream-ordered upload from pinned host memory (address `host_ptr`), then ghost fill."""
    _check(_lib.chemora_upload_state(h, _vp(host_ptr), stream), "chemora_upload_state")


def chemora_download_state(h, host_ptr: int, stream=None):
    """Stream-ordered download to pinned host memory (address `host_ptr`); no synchronisation."""
    _check(_lib.chemora_download_state(h, _vp(host_ptr), stream), "chemora_download_state")


def chemora_rhs(h, dev_dst_ptr: int, stream=None):
    _check(_lib.chemora_rhs(h, _vp(dev_dst_ptr), stream), "chemora_rhs")


def chemora_rk4_step(h, dt: float, nsteps: int, stream=None):
    _check(_lib.chemora_rk4_step(h, dt, nsteps, stream), "chemora_rk4_step")


def chemora_rk4_step_multi(handles, dt: float, nsteps: int, stream=None):
    arr = (_vp * len(handles))(*handles)
    _check(_lib.chemora_rk4_step_multi(arr, len(handles), dt, nsteps, stream), "chemora_rk4_step_multi")


def chemora_halo_exchange(h, stream=None):
    _check(_lib.chemora_halo_exchange(h, stream), "chemora_halo_exchange")


def chemora_halo_exchange_multi(handles, stream=None):
    arr = (_vp * len(handles))(*handles)
    _check(_lib.chemora_halo_exchange_multi(arr, len(handles), stream), "chemora_halo_exchange_multi")


def chemora_norms_len(system: int) -> int:
    return _lib.chemora_norms_len(system, N_GF[system])


def chemora_norms_partial(h, system, stream=None, allow_nonfinite=False) -> np.ndarray:
    out = np.zeros(chemora_norms_len(system))
    rc = _lib.chemora_norms_partial(h, _dptr(out), stream)
    if not (rc == E_NONFINITE and allow_nonfinite):
        _check(rc, "chemora_norms_partial")
    return out


def chemora_norms_combine(desc, partials: np.ndarray, nranks: int) -> np.ndarray:
    partials = np.ascontiguousarray(partials, dtype=np.float64)
    out = np.zeros(chemora_norms_len(desc.system))
    _check(_lib.chemora_norms_combine(ctypes.byref(desc), _dptr(partials), nranks, _dptr(out)),
           "chemora_norms_combine")
    return out


def chemora_norms(h, system, stream=None) -> np.ndarray:
    out = np.zeros(chemora_norms_len(system))
    _check(_lib.chemora_norms(h, _dptr(out), stream), "chemora_norms")
    return out


def chemora_constraints(h, dev_fields_ptr: int | None = None, partials: bool = True, stream=None):
    """BSSN constraint fields into a device buffer (optional) and/or the 14 local partials
    [sum c_q^2, max |c_q|] x (H, M1..3, G1..3)."""
    out = np.zeros(14) if partials else None
    _check(_lib.chemora_constraints(h, _vp(dev_fields_ptr) if dev_fields_ptr else None, _dptr(out), stream),
           "chemora_constraints")
    return out


def chemora_constraint_norms(h, stream=None) -> np.ndarray:
    out = np.zeros(14)
    _check(_lib.chemora_constraint_norms(h, _dptr(out), stream), "chemora_constraint_norms")
    return out


def chemora_grid_connect_local(handles):
    arr = (_vp * len(handles))(*handles)
    _check(_lib.chemora_grid_connect_local(arr, len(handles)), "chemora_grid_connect_local")


def chemora_peer_record_size() -> int:
    n = ctypes.c_size_t()
    _check(_lib.chemora_peer_record_size(ctypes.byref(n)), "chemora_peer_record_size")
    return n.value


def chemora_grid_export_peer(h) -> bytes:
    buf = ctypes.create_string_buffer(chemora_peer_record_size())
    _check(_lib.chemora_grid_export_peer(h, buf), "chemora_grid_export_peer")
    return buf.raw


def chemora_grid_connect_ipc(h, rec_lo: bytes, rec_hi: bytes):
    _check(_lib.chemora_grid_connect_ipc(h, ctypes.c_char_p(rec_lo), ctypes.c_char_p(rec_hi)),
           "chemora_grid_connect_ipc")


def chemora_set_kernel_variant(h, variant: int):
    _check(_lib.chemora_set_kernel_variant(h, variant), "chemora_set_kernel_variant")


def chemora_set_monitor(h, enable: bool):
    _check(_lib.chemora_set_monitor(h, 1 if enable else 0), "chemora_set_monitor")


def chemora_read_monitor(h, max_steps: int = 1024, stream=None, width: int = 1) -> np.ndarray:
    """Per-step monitor values since the last read: width 1 (wave energies) -> shape (n,);
    width 14 (BSSN [L2, Linf] x (H, M1..3, G1..3)) -> shape (n, 14)."""
    out = np.zeros(max(1, max_steps) * width)
    cnt = ctypes.c_int32()
    _check(_lib.chemora_read_monitor(h, _dptr(out), max_steps, ctypes.byref(cnt), stream),
           "chemora_read_monitor")
    out = out[:cnt.value * width].copy()
    return out if width == 1 else out.reshape(cnt.value, width)


def chemora_read_monitor_multi(handles, max_steps: int = 1024, stream=None, width: int = 1) -> np.ndarray:
    arr = (_vp * len(handles))(*handles)
    out = np.zeros(max(1, max_steps) * width)
    cnt = ctypes.c_int32()
    _check(_lib.chemora_read_monitor_multi(arr, len(handles), _dptr(out), max_steps, ctypes.byref(cnt), stream),
           "chemora_read_monitor_multi")
    out = out[:cnt.value * width].copy()
    return out if width == 1 else out.reshape(cnt.value, width)


def chemora_set_launch_timing(h, enable: bool):
    _check(_lib.chemora_set_launch_timing(h, 1 if enable else 0), "chemora_set_launch_timing")


def chemora_read_launch_timing(h, stream=None):
    """-> (ms_sum[8], counts[8]) per launch slot since the last read."""
    ms = np.zeros(8)
    cnt = (ctypes.c_int32 * 8)()
    _check(_lib.chemora_read_launch_timing(h, _dptr(ms), cnt, stream), "chemora_read_launch_timing")
    return ms, list(cnt)


BARRIER_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p)


def chemora_set_phase_barrier(h, fn):
    """fn: a BARRIER_FN (keep a reference alive while the handle uses it) or None."""
    _check(_lib.chemora_set_phase_barrier(h, ctypes.cast(fn, _vp) if fn is not None else None, None),
           "chemora_set_phase_barrier")


def chemora_constraint_norms_combine(desc, partials: np.ndarray, nranks: int) -> np.ndarray:
    partials = np.ascontiguousarray(partials, dtype=np.float64)
    out = np.zeros(14)
    _check(_lib.chemora_constraint_norms_combine(ctypes.byref(desc), _dptr(partials), nranks, _dptr(out)),
           "chemora_constraint_norms_combine")
    return out


def chemora_autotune(h, trials: int = 3, stream=None):
    chosen = (ctypes.c_int32 * 3)()
    ms = np.zeros(4)
    _check(_lib.chemora_autotune(h, trials, chosen, _dptr(ms), stream), "chemora_autotune")
    return {"variant": chosen[0], "band": chosen[1], "candidates": chosen[2],
            "ms": ms[:chosen[2]].tolist()}

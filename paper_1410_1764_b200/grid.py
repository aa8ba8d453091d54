"""User-facing Python handle over the C ABI: PyTorch supplies the device workspace, the
stream and (for multi-process runs) the process group; everything else is a call into
``libchemora.so`` (see capi.py and include/chemora.h)."""
from __future__ import annotations

import numpy as np
import torch

from . import capi as C
from . import dist as D


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class Grid:
    """One z-slab (or the whole periodic grid when ``nranks == 1``) on one device."""

    def __init__(self, system, extent, spacing, origin=(0.0, 0.0, 0.0), ghost=3, device=0,
                 rank=0, nranks=1, fd_order=0, params=None):
        self.system = system
        self.device = torch.device("cuda", device)
        self.desc = C.make_desc(system, extent, spacing, origin, ghost, device, rank, nranks,
                                fd_order, params)
        self.nbytes = C.chemora_grid_required_bytes(self.desc)
        self.workspace = torch.empty(self.nbytes, dtype=torch.uint8, device=self.device)
        self.handle = C.chemora_grid_create(self.desc, self.workspace.data_ptr(), self.nbytes)
        self.local_extent, self.z0 = C.chemora_grid_local(self.handle)
        self.n_gf = C.N_GF[system]
        self.ghost = ghost
        self.rank, self.nranks = rank, nranks

    # ---------------------------------------------------------------- helpers
    @property
    def stream(self):
        return _stream_ptr(self.device)

    def interior_shape(self):
        nx, ny, nz = self.local_extent
        return (self.n_gf, nz, ny, nx)

    def padded_shape(self):
        nx, ny, nz = self.local_extent
        g = self.ghost
        return (self.n_gf, nz + 2 * g, ny + 2 * g, nx + 2 * g)

    # ---------------------------------------------------------------- API
    def set_initial(self, kind, host=None, kind_params=None, seed=0, fill=True):
        C.chemora_set_initial(self.handle, kind, host, kind_params, seed, self.stream, fill)

    def get_state(self, padded=False, out=None, allow_nonfinite=False):
        shape = self.padded_shape() if padded else self.interior_shape()
        if out is None:
            out = np.empty(shape)
        C.chemora_get_state(self.handle, out, self.stream, padded, allow_nonfinite)
        return out

    def upload_state(self, host: torch.Tensor):
        """Enqueue the upload of a pinned host tensor [gf][z][y][x] on this grid's stream."""
        assert host.is_pinned() and host.dtype == torch.float64 and host.is_contiguous()
        assert tuple(host.shape) == self.interior_shape()
        C.chemora_upload_state(self.handle, host.data_ptr(), self.stream)

    def download_state(self, host: torch.Tensor):
        """Enqueue the download into a pinned host tensor on this grid's stream (no sync)."""
        assert host.is_pinned() and host.dtype == torch.float64 and host.is_contiguous()
        assert tuple(host.shape) == self.interior_shape()
        C.chemora_download_state(self.handle, host.data_ptr(), self.stream)

    def rhs(self, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.empty(self.interior_shape(), dtype=torch.float64, device=self.device)
        assert out.is_contiguous() and out.dtype == torch.float64
        C.chemora_rhs(self.handle, out.data_ptr(), self.stream)
        return out

    def rk4_step(self, dt, nsteps=1):
        C.chemora_rk4_step(self.handle, dt, nsteps, self.stream)

    def halo_exchange(self):
        C.chemora_halo_exchange(self.handle, self.stream)

    def norms(self):
        """Global norms (collective over the IPC-connected slabs when nranks > 1)."""
        return C.chemora_norms(self.handle, self.system, self.stream)

    def constraints(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """BSSN constraint fields [H, M1, M2, M3, G1, G2, G3][z][y][x] of the current state."""
        if out is None:
            n = self.interior_shape()
            out = torch.empty((7,) + tuple(n[1:]), dtype=torch.float64, device=self.device)
        assert out.is_contiguous() and out.dtype == torch.float64
        C.chemora_constraints(self.handle, out.data_ptr(), False, self.stream)
        return out

    def constraint_norms(self) -> np.ndarray:
        """[L2, Linf] of H, M1..3, G1..3 (14 doubles), over all ranks (collective)."""
        return C.chemora_constraint_norms(self.handle, self.stream)

    def connect_ipc(self, group=None, host_barrier=False):
        """Exchange peer records over torch.distributed and open the ring neighbours.
        host_barrier: end every phase with a stream sync + torch.distributed barrier
        (chemora_set_phase_barrier) -- required when ranks share one device."""
        rec = C.chemora_grid_export_peer(self.handle)
        lo, hi = D.exchange_records(rec, self.rank, self.nranks, group)
        C.chemora_grid_connect_ipc(self.handle, lo, hi)
        if host_barrier:
            self._barrier = C.BARRIER_FN(D.barrier_callback(group))
            C.chemora_set_phase_barrier(self.handle, self._barrier)

    def set_kernel_variant(self, v):
        C.chemora_set_kernel_variant(self.handle, v)

    def kernel_variant(self) -> int:
        v = C.ctypes.c_int()
        C._check(C._lib.chemora_get_kernel_variant(self.handle, C.ctypes.byref(v)), "chemora_get_kernel_variant")
        return v.value

    def set_monitor(self, enable=True):
        C.chemora_set_monitor(self.handle, enable)

    def read_monitor(self, max_steps=1024):
        """Per-step monitor values since the last read (global values, collective when
        nranks > 1): wave -- the energy after each step, shape (n,); BSSN -- [L2, Linf] of
        H, M1..3, G1..3 of the state entering each step, shape (n, 14)."""
        w = 14 if self.system == C.SYS_BSSN else 1
        return C.chemora_read_monitor(self.handle, max_steps, self.stream, w)

    def autotune(self, trials=3):
        return C.chemora_autotune(self.handle, trials, self.stream)

    def close(self):
        if getattr(self, "handle", None) is not None:
            C.chemora_grid_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalSlabs:
    """The z-slab decomposition emulated on ONE device: P slab handles in this process,
    connected so every stage kernel stores its boundary planes straight into the
    neighbouring slab's ghost planes, stepped stage-interleaved on one stream."""

    def __init__(self, system, extent, spacing, nslabs, origin=(0.0, 0.0, 0.0), ghost=3,
                 device=0, fd_order=0, params=None):
        self.grids = [Grid(system, extent, spacing, origin, ghost, device, r, nslabs, fd_order, params)
                      for r in range(nslabs)]
        self.handles = [g.handle for g in self.grids]
        C.chemora_grid_connect_local(self.handles)
        self.nslabs = nslabs

    @property
    def stream(self):
        return self.grids[0].stream

    def set_initial(self, kind, host=None, kind_params=None, seed=0):
        for g in self.grids:
            src = None
            if host is not None:
                nz = g.local_extent[2]
                src = np.ascontiguousarray(host[:, g.z0:g.z0 + nz])
            g.set_initial(kind, src, kind_params, seed, fill=False)
        C.chemora_halo_exchange_multi(self.handles, self.stream)

    def rk4_step(self, dt, nsteps=1):
        C.chemora_rk4_step_multi(self.handles, dt, nsteps, self.stream)

    def get_state(self):
        return np.concatenate([g.get_state() for g in self.grids], axis=1)

    def get_state_padded(self):
        return [g.get_state(padded=True) for g in self.grids]

    def norms(self):
        parts = np.array([C.chemora_norms_partial(g.handle, g.system, self.stream) for g in self.grids])
        return C.chemora_norms_combine(self.grids[0].desc, parts, self.nslabs)

    def set_monitor(self, enable=True):
        for g in self.grids:
            C.chemora_set_monitor(g.handle, enable)

    def read_monitor(self, max_steps=1024):
        """Per-step global energies: the slabs' fused-monitor values summed in slab order."""
        w = 14 if self.grids[0].system == C.SYS_BSSN else 1
        return C.chemora_read_monitor_multi(self.handles, max_steps, self.stream, w)

    def close(self):
        for g in self.grids:
            g.close()

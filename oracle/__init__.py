"""ctypes front end of the CPU oracle (oracle/chemora_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs -- never by the product package
``paper_1410_1764_b200``.  See the header of chemora_oracle.cpp for what each function
computes and which passage of the paper it follows.

Array conventions: ``interior`` arrays are ``[gf][Nz][Ny][Nx]`` float64; ``padded`` arrays
are ``[gf][Nz+2g][Ny+2g][Nx+2g]``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "chemora_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
WAVE, BSSN = 1, 2
N_GF = {WAVE: 5, BSSN: 25}
DEFAULT_GHOST = 3

_LIB_FMA = os.path.join(_HERE, "liboracle_fma.so")
_libs = {}


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++ -O2 -fopenmp -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def build_fma(force: bool = False) -> str:
    """The SAME source built with FMA contraction (-mfma -ffp-contract=fast): a second,
    equally legitimate rounding sequence of the same arithmetic.  Its difference from the
    plain build is the oracle's own rounding-noise floor, the scale
    against which GPU-vs-oracle differences at large grids are read."""
    if force or not os.path.exists(_LIB_FMA) or os.path.getmtime(_LIB_FMA) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-mfma", "-ffp-contract=fast", "-fno-fast-math",
               "-shared", "-fPIC", "-o", _LIB_FMA + ".tmp", _SRC]
        subprocess.check_call(cmd)
        os.replace(_LIB_FMA + ".tmp", _LIB_FMA)
    return _LIB_FMA


def host_has_fma() -> bool:
    try:
        with open("/proc/cpuinfo") as fh:
            return any(line.startswith("flags") and " fma " in line + " " for line in fh)
    except OSError:
        return False


class use_fma_build:
    """Context manager: oracle calls inside use the FMA-contracted build (noise floor)."""

    def __enter__(self):
        global _lib
        self._saved = _lib
        _lib = lib("fma")
        return self

    def __exit__(self, *a):
        global _lib
        _lib = self._saved


_lib = None


def lib(kind: str = ""):
    global _lib
    if kind == "" and _lib is not None:
        return _lib
    key = kind or "plain"
    if key not in _libs:
        path = build_fma() if kind == "fma" else build()
        L = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        L.chemora_oracle_fill_ghosts.argtypes = [dp, ctypes.c_int, i64p, ctypes.c_int]
        L.chemora_oracle_rhs_order.argtypes = [ctypes.c_int, dp, dp, i64p, ctypes.c_int, dp, dp,
                                               ctypes.c_int]
        L.chemora_oracle_rk4_order.argtypes = [ctypes.c_int, dp, i64p, ctypes.c_int, dp,
                                               ctypes.c_double, ctypes.c_int, dp, ctypes.c_int]
        L.chemora_oracle_norms.argtypes = [ctypes.c_int, dp, i64p, ctypes.c_int, dp, dp]
        L.chemora_oracle_default_bssn_params.argtypes = [dp]
        L.chemora_oracle_constraints.argtypes = [dp, i64p, ctypes.c_int, dp, dp]
        _libs[key] = L
    if kind == "":
        _lib = _libs[key]
    return _libs[key]


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ext(n):
    return (ctypes.c_int64 * 3)(*[int(v) for v in n])


def _sp(h):
    return (ctypes.c_double * 3)(*[float(v) for v in h])


def _params(params):
    if params is None:
        return None
    arr = np.ascontiguousarray(params, dtype=np.float64)
    return arr


def default_bssn_params() -> np.ndarray:
    out = np.zeros(10)
    lib().chemora_oracle_default_bssn_params(_dp(out))
    return out


def extent_of(interior: np.ndarray):
    return (interior.shape[3], interior.shape[2], interior.shape[1])


def pad(interior: np.ndarray, g: int = DEFAULT_GHOST) -> np.ndarray:
    """Embed an interior array in a padded one (ghosts zero, NOT filled)."""
    nf = interior.shape[0]
    out = np.zeros((nf,) + tuple(s + 2 * g for s in interior.shape[1:]))
    out[:, g:-g, g:-g, g:-g] = interior
    return out


def unpad(padded: np.ndarray, g: int = DEFAULT_GHOST) -> np.ndarray:
    return np.ascontiguousarray(padded[:, g:-g, g:-g, g:-g])


def fill_ghosts(padded: np.ndarray, g: int = DEFAULT_GHOST) -> np.ndarray:
    """Periodic ghost fill in place (and returned)."""
    assert padded.dtype == np.float64 and padded.flags.c_contiguous
    n = (padded.shape[3] - 2 * g, padded.shape[2] - 2 * g, padded.shape[1] - 2 * g)
    rc = lib().chemora_oracle_fill_ghosts(_dp(padded), padded.shape[0], _ext(n), g)
    if rc:
        raise ValueError(f"oracle fill_ghosts rc={rc}")
    return padded


def rhs_padded(system: int, padded: np.ndarray, spacing, params=None,
               g: int = DEFAULT_GHOST, order: int = 4) -> np.ndarray:
    """k = F(y) on the interior, ghosts of ``padded`` used as they are."""
    padded = np.ascontiguousarray(padded, dtype=np.float64)
    n = (padded.shape[3] - 2 * g, padded.shape[2] - 2 * g, padded.shape[1] - 2 * g)
    k = np.zeros((padded.shape[0], n[2], n[1], n[0]))
    p = _params(params)
    rc = lib().chemora_oracle_rhs_order(system, _dp(padded), _dp(k), _ext(n), g, _sp(spacing),
                                        _dp(p) if p is not None else None, order)
    if rc:
        raise ValueError(f"oracle rhs rc={rc}")
    return k


def rhs(system: int, interior: np.ndarray, spacing, params=None, g: int = DEFAULT_GHOST,
        order: int = 4):
    """k = F(y) on a periodic grid (ghosts filled first).  ``order``: wave D1 accuracy."""
    p = fill_ghosts(pad(interior, g), g)
    return rhs_padded(system, p, spacing, params, g, order)


def rk4(system: int, interior: np.ndarray, spacing, dt: float, nsteps: int, params=None,
        g: int = DEFAULT_GHOST, order: int = 4) -> np.ndarray:
    """``nsteps`` textbook RK4 steps on a periodic grid; returns the new interior."""
    y = pad(np.ascontiguousarray(interior, dtype=np.float64), g)
    n = extent_of(interior)
    p = _params(params)
    rc = lib().chemora_oracle_rk4_order(system, _dp(y), _ext(n), g, _sp(spacing), float(dt),
                                        int(nsteps), _dp(p) if p is not None else None, order)
    if rc:
        raise ValueError(f"oracle rk4 rc={rc}")
    return unpad(y, g)


def norms(system: int, interior: np.ndarray, spacing, g: int = DEFAULT_GHOST) -> np.ndarray:
    """Per GF (L2, Linf, sum) then, for the wave system, the energy."""
    y = pad(np.ascontiguousarray(interior, dtype=np.float64), g)
    n = extent_of(interior)
    nf = interior.shape[0]
    out = np.zeros(3 * nf + (1 if system == WAVE else 0))
    rc = lib().chemora_oracle_norms(system, _dp(y), _ext(n), g, _sp(spacing), _dp(out))
    if rc:
        raise ValueError(f"oracle norms rc={rc}")
    return out


CONSTRAINT_NAMES = ("H", "M1", "M2", "M3", "G1", "G2", "G3")


def constraints_padded(padded: np.ndarray, spacing, g: int = DEFAULT_GHOST) -> np.ndarray:
    """BSSN constraint fields at interior points, ghosts of ``padded`` used as they are."""
    padded = np.ascontiguousarray(padded, dtype=np.float64)
    n = (padded.shape[3] - 2 * g, padded.shape[2] - 2 * g, padded.shape[1] - 2 * g)
    out = np.zeros((7, n[2], n[1], n[0]))
    rc = lib().chemora_oracle_constraints(_dp(padded), _ext(n), g, _sp(spacing), _dp(out))
    if rc:
        raise ValueError(f"oracle constraints rc={rc}")
    return out


def constraints(interior: np.ndarray, spacing, g: int = DEFAULT_GHOST) -> np.ndarray:
    """BSSN constraint fields [H, M1..3, G1..3] on a periodic grid, shape [7][Nz][Ny][Nx]."""
    y = fill_ghosts(pad(np.ascontiguousarray(interior, dtype=np.float64), g), g)
    n = extent_of(interior)
    out = np.zeros((7, n[2], n[1], n[0]))
    rc = lib().chemora_oracle_constraints(_dp(y), _ext(n), g, _sp(spacing), _dp(out))
    if rc:
        raise ValueError(f"oracle constraints rc={rc}")
    return out

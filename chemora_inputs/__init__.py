"""Seeded synthetic inputs shared by the CPU oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no stencils, no RHS, no Runge-Kutta):
only the initial-data recipes of DESIGN.md §"Input recipe" so that both sides of every
parity test start from byte-identical host arrays.

Layout of every array returned here: interior points only, ``[gf][z][y][x]`` (x fastest),
float64, global interior index ``I = i + Nx*(j + Ny*k)``.

Recipes (SURVEY.md §8(c) "Seeded inputs"; Fig. 1 ``Init``):

* ``noise``     every GF = SplitMix64 hash of (seed, gf, I) mapped to uniform [-1, 1).
* ``pw3``       three exact plane-wave solutions of Eq. 1 superposed.
* ``gaussian``  Fig. 1 Init: rho = A exp(-1/2 (r/W)^2), u = v_i = 0, r from the domain centre.
* ``polynomial`` padded (ghosts included, not periodic) polynomial data for exactness tests.
* ``mink_pert`` BSSN flat data + seeded smooth sines (SURVEY.md §8(c) MINK_PERT).
* ``gauge_wave`` BSSN gauge-wave exact data.

The same SplitMix64 counter generator is implemented (independently) in the CUDA init
kernel so large benchmark grids can be generated on the device; the GPU tests check the
two bit for bit.
"""
from __future__ import annotations

import math

import numpy as np

WAVE_GF = ("u", "rho", "v1", "v2", "v3")
BSSN_GF = ("phi", "gt11", "gt12", "gt13", "gt22", "gt23", "gt33", "trK",
           "At11", "At12", "At13", "At22", "At23", "At33",
           "Xt1", "Xt2", "Xt3", "alpha", "A", "beta1", "beta2", "beta3",
           "B1", "B2", "B3")

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser (Steele, Lea, Flood 2014) on uint64 arrays (wrapping)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def hash_uniform(seed: int, gf: int, index: np.ndarray) -> np.ndarray:
    """Uniform [-1, 1) from (seed, gf, I): ((z >> 11) * 2^-52) - 1, exact in fp64."""
    key = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (
        (np.uint64(gf) << np.uint64(40)) + np.asarray(index, dtype=np.uint64))
    z = splitmix64(key)
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0


def coords(n, spacing, origin=(0.0, 0.0, 0.0)):
    """x_i = origin + i*h; returns broadcastable (z, y, x) grids."""
    nx, ny, nz = n
    x = origin[0] + np.arange(nx) * spacing[0]
    y = origin[1] + np.arange(ny) * spacing[1]
    z = origin[2] + np.arange(nz) * spacing[2]
    return z[:, None, None], y[None, :, None], x[None, None, :]


def noise_box(gext, n_gf, seed, lo, size):
    """NOISE values on the box [lo, lo+size) of a periodic global grid of extents ``gext``
    (indices wrap), so a sample of a huge grid can be regenerated on the host."""
    nx, ny, nz = gext
    i = (np.arange(lo[0], lo[0] + size[0]) % nx).astype(np.uint64)[None, None, :]
    j = (np.arange(lo[1], lo[1] + size[1]) % ny).astype(np.uint64)[None, :, None]
    k = (np.arange(lo[2], lo[2] + size[2]) % nz).astype(np.uint64)[:, None, None]
    index = i + np.uint64(nx) * (j + np.uint64(ny) * k)
    out = np.empty((n_gf, size[2], size[1], size[0]))
    for g in range(n_gf):
        out[g] = hash_uniform(seed, g, index)
    return out


def noise(n, n_gf, seed, z0=0, nz_global=None):
    """Uniform [-1,1) noise on every GF keyed by the GLOBAL index.

    ``z0`` / ``nz_global`` select a z-slab of a larger global grid (multi-rank).
    """
    nx, ny, nz = n
    k = np.arange(z0, z0 + nz, dtype=np.uint64)[:, None, None]
    j = np.arange(ny, dtype=np.uint64)[None, :, None]
    i = np.arange(nx, dtype=np.uint64)[None, None, :]
    index = i + np.uint64(nx) * (j + np.uint64(ny) * k)
    out = np.empty((n_gf, nz, ny, nx))
    for g in range(n_gf):
        out[g] = hash_uniform(seed, g, index)
    return out


# Plane-wave modes for PW3: wave vectors, amplitudes, phases.
PW3_MODES = (((1, 2, 3), 1.0, 0.0), ((2, -1, 1), 0.5, 0.3), ((0, 1, -2), 0.25, 1.1))


def pw3(n, spacing, origin=(0.0, 0.0, 0.0), t=0.0, modes=PW3_MODES):
    """Superposed continuum plane waves u = sum a sin(k.x - |k| t + phi) of Eq. 1.

    rho = du/dt, v_i = du/dx_i, so each mode is an exact solution of PAPER.md:320-327.
    """
    z, y, x = coords(n, spacing, origin)
    out = np.zeros((5,) + (n[2], n[1], n[0]))
    for (kx, ky, kz), a, ph in modes:
        w = math.sqrt(kx * kx + ky * ky + kz * kz)
        arg = kx * x + ky * y + kz * z - w * t + ph
        s, c = np.sin(arg), np.cos(arg)
        out[0] += a * s
        out[1] += -a * w * c
        out[2] += a * kx * c
        out[3] += a * ky * c
        out[4] += a * kz * c
    return out


def gaussian(n, spacing, origin=(0.0, 0.0, 0.0), amplitude=1.0, width=0.5):
    """Fig. 1 ``Init``: u = 0, rho = A exp(-1/2 (r/W)^2), v_i = 0.

    r is the distance to the domain centre."""
    z, y, x = coords(n, spacing, origin)
    c = [origin[a] + 0.5 * n[a] * spacing[a] for a in range(3)]
    r2 = (x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2
    out = np.zeros((5, n[2], n[1], n[0]))
    out[1] = amplitude * np.exp(-0.5 * r2 / (width * width))
    return out


def padded_coords(n, g, spacing, origin=(0.0, 0.0, 0.0)):
    """Coordinates of the padded grid (ghosts included, NOT wrapped)."""
    nx, ny, nz = n
    x = origin[0] + np.arange(-g, nx + g) * spacing[0]
    y = origin[1] + np.arange(-g, ny + g) * spacing[1]
    z = origin[2] + np.arange(-g, nz + g) * spacing[2]
    return z[:, None, None], y[None, :, None], x[None, None, :]


def random_polynomial_coeffs(rng: np.random.Generator, degree: int):
    """Random integer coefficients c[a,b,c] of x^a y^b z^c with a+b+c <= degree."""
    out = {}
    for a in range(degree + 1):
        for b in range(degree + 1 - a):
            for c in range(degree + 1 - a - b):
                out[(a, b, c)] = float(rng.integers(-3, 4))
    return out


def eval_polynomial(coeffs, x, y, z):
    val = 0.0
    for (a, b, c), w in coeffs.items():
        val = val + w * x ** a * y ** b * z ** c
    return val


def mink_pert(n, spacing, seed, eps=1e-3, origin=(0.0, 0.0, 0.0), n_modes=2, kmax=2,
              length=None):
    """BSSN perturbed Minkowski data (SURVEY.md §8(c) MINK_PERT).

    Flat values (gt_ii = alpha = 1, all else 0) plus, on every GF,
    eps * sum_m c_m sin(2 pi n_m . x / L + phi_m) with integer n_m in [-kmax, kmax]^3 \\ 0,
    phi_m in [0, 2 pi), c_m in [1/2, 1), all drawn from hash(seed, gf, m)."""
    z, y, x = coords(n, spacing, origin)
    if length is None:
        length = n[0] * spacing[0]
    out = np.zeros((25, n[2], n[1], n[0]))
    for name in ("gt11", "gt22", "gt33", "alpha"):
        out[BSSN_GF.index(name)] = 1.0
    span = 2 * kmax + 1
    for g in range(25):
        for m in range(n_modes):
            draws = hash_uniform(seed, 1000 + g, np.arange(8 * m, 8 * m + 8, dtype=np.uint64))
            u = (draws + 1.0) * 0.5  # [0,1)
            kv = [int(min(span - 1, math.floor(u[a] * span))) - kmax for a in range(3)]
            if kv == [0, 0, 0]:
                kv = [1, 0, 0]
            phase = 2 * math.pi * u[3]
            amp = 0.5 + 0.5 * u[4]
            arg = 2 * math.pi * (kv[0] * x + kv[1] * y + kv[2] * z) / length + phase
            out[g] += eps * amp * np.sin(arg)
    return out


def gauge_wave(n, spacing, t=0.0, amp=0.1, d=1.0, shift=0.0, origin=(0.0, 0.0, 0.0)):
    """Gauge-wave exact data at time t, optionally with a constant
    shift beta^x = ``shift`` (the shifted gauge wave, solution f(x + v t, t))."""
    z, y, x = coords(n, spacing, origin)
    xs = x + shift * t
    ph = 2 * math.pi * (xs - t) / d
    H = 1.0 - amp * np.sin(ph)
    dHdt = amp * (2 * math.pi / d) * np.cos(ph)
    dHdx = -amp * (2 * math.pi / d) * np.cos(ph)
    shape = (n[2], n[1], n[0])
    out = np.zeros((25,) + shape)

    def put(name, val):
        out[BSSN_GF.index(name)] = np.broadcast_to(val, shape)

    Kxx = -dHdt / (2 * np.sqrt(H))
    put("phi", np.log(H) / 12.0)
    put("gt11", H ** (2.0 / 3.0))
    put("gt22", H ** (-1.0 / 3.0))
    put("gt33", H ** (-1.0 / 3.0))
    put("trK", Kxx / H)
    put("At11", (2.0 / 3.0) * H ** (-1.0 / 3.0) * Kxx)
    put("At22", -(1.0 / 3.0) * H ** (-4.0 / 3.0) * Kxx)
    put("At33", -(1.0 / 3.0) * H ** (-4.0 / 3.0) * Kxx)
    put("Xt1", (2.0 / 3.0) * H ** (-5.0 / 3.0) * dHdx)
    put("alpha", np.sqrt(H))
    put("beta1", shift)
    return out

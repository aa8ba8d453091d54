"""Independent mathematical pins used by the oracle tests (no oracle code here).

* exact rational moment solve for finite-difference coefficients (SPEC.md:191-194, 246:
  sum_k c_k k^m = d! [m == d] for m = 0 .. len(offsets)-1)
* the fully discrete Fourier symbol of the 4th-order wave scheme and the RK4 amplification
  polynomial, giving a closed-form solution of the discrete scheme.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np


def moment_solve(deriv_order: int, offsets) -> list[Fraction]:
    """Coefficients c_k on ``offsets`` with sum_k c_k k^m = d! [m == d], exact rationals.

    Gaussian elimination over Fractions of the len(offsets) x len(offsets) Vandermonde
    system (rows m = 0..n-1)."""
    offs = [Fraction(o) for o in offsets]
    n = len(offs)
    A = [[o ** m for o in offs] + [Fraction(math.factorial(deriv_order) if m == deriv_order else 0)]
         for m in range(n)]
    for col in range(n):
        piv = next(r for r in range(col, n) if A[r][col] != 0)
        A[col], A[piv] = A[piv], A[col]
        p = A[col][col]
        A[col] = [v / p for v in A[col]]
        for r in range(n):
            if r != col and A[r][col] != 0:
                f = A[r][col]
                A[r] = [a - f * b for a, b in zip(A[r], A[col])]
    return [A[r][n] for r in range(n)]


def read_golden_stencils(path):
    rows = []
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            left, right = line.split(":")
            nums = [int(v) for v in left.split()]
            d, w, offs = nums[0], nums[1], nums[2:]
            coeffs = [Fraction(v) for v in right.split()]
            rows.append((d, w, offs, coeffs))
    return rows


def rk4_poly(Z: np.ndarray) -> np.ndarray:
    """P(Z) = I + Z + Z^2/2 + Z^3/6 + Z^4/24 (classical RK4 on a linear system)."""
    I = np.eye(Z.shape[0], dtype=complex)
    Z2 = Z @ Z
    Z3 = Z2 @ Z
    Z4 = Z3 @ Z
    return I + Z + Z2 / 2 + Z3 / 6 + Z4 / 24


def wave_symbol(kvec, h) -> np.ndarray:
    """5x5 symbol M of the semi-discrete 4th-order wave scheme for the mode e^{i k.x}.

    D1 e^{ikx} = i ktilde e^{ikx} with ktilde = (8 sin kh - sin 2kh) / (6h); state order
    (u, rho, v1, v2, v3); M[u,rho] = 1, M[rho,v_j] = M[v_j,rho] = i ktilde_j."""
    kt = [(8 * math.sin(k * hh) - math.sin(2 * k * hh)) / (6 * hh) for k, hh in zip(kvec, h)]
    M = np.zeros((5, 5), dtype=complex)
    M[0, 1] = 1.0
    for j in range(3):
        M[1, 2 + j] = 1j * kt[j]
        M[2 + j, 1] = 1j * kt[j]
    return M


def discrete_plane_wave(n, h, dt, nsteps, modes):
    """Exact solution of the fully discrete scheme (4th-order FD + RK4) for PW3-type data.

    Each mode u = a sin(k.x + phi), rho = -a|k| cos, v_j = a k_j cos is written as
    Re(c e^{i k.x}) with c = e^{i phi} (-i a, -a|k|, a kx, a ky, a kz) and advanced by
    P(dt M)^nsteps."""
    nx, ny, nz = n
    x = np.arange(nx)[None, None, :] * h[0]
    y = np.arange(ny)[None, :, None] * h[1]
    z = np.arange(nz)[:, None, None] * h[2]
    out = np.zeros((5, nz, ny, nx))
    for (kx, ky, kz), a, ph in modes:
        w = math.sqrt(kx * kx + ky * ky + kz * kz)
        c = np.exp(1j * ph) * np.array([-1j * a, -a * w, a * kx, a * ky, a * kz], dtype=complex)
        P = rk4_poly(dt * wave_symbol((kx, ky, kz), h))
        cn = np.linalg.matrix_power(P, nsteps) @ c
        e = np.exp(1j * (kx * x + ky * y + kz * z))
        for f in range(5):
            out[f] += (cn[f] * e).real
    return out


def ktilde(k: float, h: float, order: int) -> float:
    """Fourier symbol of the centered D1 of accuracy ``order``: D1 e^{ikx} = i ktilde e^{ikx},
    ktilde = sum_{s>0} 2 c_s sin(s k h) / h with c_s from the exact moment solve."""
    w = order // 2
    c = moment_solve(1, range(-w, w + 1))
    return sum(2.0 * float(c[w + s]) * math.sin(s * k * h) for s in range(1, w + 1)) / h


def discrete_plane_wave_order(n, h, dt, nsteps, modes, order):
    """discrete_plane_wave for a centered D1 of any even accuracy order."""
    nx, ny, nz = n
    x = np.arange(nx)[None, None, :] * h[0]
    y = np.arange(ny)[None, :, None] * h[1]
    z = np.arange(nz)[:, None, None] * h[2]
    out = np.zeros((5, nz, ny, nx))
    for (kx, ky, kz), a, ph in modes:
        w = math.sqrt(kx * kx + ky * ky + kz * kz)
        c = np.exp(1j * ph) * np.array([-1j * a, -a * w, a * kx, a * ky, a * kz], dtype=complex)
        M = np.zeros((5, 5), dtype=complex)
        M[0, 1] = 1.0
        for j, (kk, hh) in enumerate(zip((kx, ky, kz), h)):
            M[1, 2 + j] = M[2 + j, 1] = 1j * ktilde(kk, hh, order)
        cn = np.linalg.matrix_power(rk4_poly(dt * M), nsteps) @ c
        e = np.exp(1j * (kx * x + ky * y + kz * z))
        for f in range(5):
            out[f] += (cn[f] * e).real
    return out

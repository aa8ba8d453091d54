"""Pins of the CPU oracle's wave path against what the paper and the mathematics fix.

Each test names the plausible oracle mistake it would catch.
"""
from __future__ import annotations

import math
import os
from fractions import Fraction

import numpy as np
import pytest

import chemora_inputs as ci
import oracle
from tests import pins

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "stencil_coefficients.txt")
W = oracle.WAVE


# ------------------------------------------------------------------ stencil coefficients
def test_moment_solve_matches_printed_coefficients():
    """The exact moment solve reproduces every coefficient printed in the paper/SPEC
    (SPEC.md:216-218).  Pins the pin itself."""
    rows = pins.read_golden_stencils(GOLDEN)
    assert len(rows) == 3
    for d, w, offs, coeffs in rows:
        assert pins.moment_solve(d, offs) == coeffs


def test_moment_solve_derived_stencils():
    """4th-order D2, lopsided upwind D+/D- and the S/A split."""
    assert pins.moment_solve(2, range(-2, 3)) == [Fraction(v, 12) for v in (-1, 16, -30, 16, -1)]
    assert pins.moment_solve(1, range(-1, 4)) == [Fraction(v, 12) for v in (-3, -10, 18, -6, 1)]
    assert pins.moment_solve(1, range(-3, 2)) == [Fraction(v, 12) for v in (-1, 6, -18, 10, 3)]
    dp = [Fraction(0)] * 2 + pins.moment_solve(1, range(-1, 4))
    dm = pins.moment_solve(1, range(-3, 2)) + [Fraction(0)] * 2
    S = [(a + b) / 2 for a, b in zip(dp, dm)]
    A = [(a - b) / 2 for a, b in zip(dp, dm)]
    assert S == [Fraction(v, 24) for v in (-1, 6, -21, 0, 21, -6, 1)]
    assert A == [Fraction(v, 24) for v in (1, -6, 15, -20, 15, -6, 1)]


def _oracle_d1_weights(axis: int, h: float):
    """Read the oracle's D1 stencil weights off its wave RHS applied to a delta function.

    d_t v_axis = D_axis rho, so with rho = delta at p the output at p - s is c_s / h."""
    n = (12, 12, 12)
    y = np.zeros((5, 12, 12, 12))
    y[1, 6, 6, 6] = 1.0
    k = oracle.rhs(W, y, (h, h, h))
    line = []
    for s in range(-3, 4):
        idx = [6, 6, 6]  # z, y, x
        idx[2 - axis] -= s
        line.append(k[2 + axis][tuple(idx)] * h)
    return line


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_oracle_d1_weights_are_the_moment_solution(axis):
    """Catches a wrong/dropped stencil coefficient, sign or axis in the oracle RHS."""
    h = 0.375
    got = _oracle_d1_weights(axis, h)
    exact = [0.0] + [float(c) for c in pins.moment_solve(1, range(-2, 3))] + [0.0]
    np.testing.assert_allclose(got, exact, rtol=1e-15, atol=1e-15)


def test_oracle_rho_rhs_weights():
    """d_t rho = D1x v1 + D1y v2 + D1z v3 (Eq. 1): each v_j enters only along its axis."""
    h = 0.5
    exact = [float(c) for c in pins.moment_solve(1, range(-2, 3))]
    for j in range(3):
        y = np.zeros((5, 10, 10, 10))
        y[2 + j, 5, 5, 5] = 1.0
        k = oracle.rhs(W, y, (h, h, h))
        nz = np.argwhere(k[1] != 0.0)
        assert len(nz) == 4
        for s, c in zip(range(-2, 3), exact):
            idx = [5, 5, 5]
            idx[2 - j] -= s
            assert k[1][tuple(idx)] * h == pytest.approx(c, rel=1e-15, abs=1e-15)
        assert np.all(k[[0, 2, 3, 4]] == 0.0)


# ------------------------------------------------------------------ polynomial exactness
@pytest.mark.parametrize("degree", [0, 1, 2, 3, 4])
def test_polynomial_exactness(degree):
    """On non-periodic polynomial data (ghosts = polynomial values, HOST_PADDED) the FD
    RHS equals the continuum RHS of Eq. 1 exactly for degree <= 4 (D1 is 4th order)."""
    rng = np.random.default_rng(100 + degree)
    g, n, h = 3, (7, 6, 8), (0.5, 0.25, 0.125)
    z, y, x = ci.padded_coords(n, g, h, origin=(-1.0, 0.5, -0.25))
    P = [ci.random_polynomial_coeffs(rng, degree) for _ in range(5)]
    pad = np.zeros((5,) + (n[2] + 2 * g, n[1] + 2 * g, n[0] + 2 * g))
    for f in range(5):
        pad[f] = ci.eval_polynomial(P[f], x, y, z)
    k = oracle.rhs_padded(W, pad, h, g=g)

    def deriv(coeffs, axis):
        out = {}
        for (a, b, c), w in coeffs.items():
            e = (a, b, c)[axis]
            if e:
                key = list((a, b, c))
                key[axis] -= 1
                out[tuple(key)] = out.get(tuple(key), 0.0) + w * e
        return out

    zi, yi, xi = z[g:-g], y[:, g:-g], x[:, :, g:-g]
    ev = lambda c: ci.eval_polynomial(c, xi, yi, zi) + np.zeros((n[2], n[1], n[0]))
    expect = [ev(P[1]),
              ev(deriv(P[2], 0)) + ev(deriv(P[3], 1)) + ev(deriv(P[4], 2)),
              ev(deriv(P[1], 0)), ev(deriv(P[1], 1)), ev(deriv(P[1], 2))]
    for f in range(5):
        np.testing.assert_allclose(k[f], expect[f], rtol=0, atol=1e-11)


def test_polynomial_degree5_is_not_exact():
    """Sensitivity check: x^5 is NOT differentiated exactly (truncation error h^4)."""
    g, n, h = 3, (8, 6, 6), (0.5, 0.5, 0.5)
    z, y, x = ci.padded_coords(n, g, h)
    pad = np.zeros((5,) + (n[2] + 2 * g, n[1] + 2 * g, n[0] + 2 * g))
    pad[1] = x ** 5 + 0 * y + 0 * z
    k = oracle.rhs_padded(W, pad, h, g=g)
    xi = x[0, 0, g:-g]
    err = k[2][0, 0, :] - 5 * xi ** 4
    # truncation error of the 4th-order D1 on x^5: -(h^4/30) * 5! = -4 h^4
    np.testing.assert_allclose(err, -4.0 * h[0] ** 4, rtol=1e-10)


# ------------------------------------------------------------------ ghost fill
def test_ghost_fill_1d_example():
    """N=4, g=1, interior [a,b,c,d] -> padded [d,a,b,c,d,a]."""
    n = (4, 4, 4)
    y = np.zeros((1, 6, 6, 6))
    y[0, 1:-1, 1:-1, 1:-1] = np.arange(64, dtype=float).reshape(4, 4, 4) + 1
    oracle.fill_ghosts(y, g=1)
    row = y[0, 2, 2, :]
    a, b, c, d = row[1:5]
    assert list(row) == [d, a, b, c, d, a]


@pytest.mark.parametrize("n,g", [((6, 7, 8), 3), ((9, 6, 6), 2), ((4, 4, 4), 2)])
def test_ghost_fill_is_modular_indexing(n, g):
    """Every padded point (edges and corners included) equals the interior value at the
    coordinates taken mod N -- compared with numpy's wrap padding."""
    rng = np.random.default_rng(7)
    interior = rng.standard_normal((2, n[2], n[1], n[0]))
    y = oracle.fill_ghosts(oracle.pad(interior, g), g)
    ref = np.pad(interior, ((0, 0), (g, g), (g, g), (g, g)), mode="wrap")
    assert np.array_equal(y, ref)


# ------------------------------------------------------------------ whole scheme
@pytest.mark.parametrize("n", [(16, 16, 16), (12, 10, 8)])
def test_discrete_plane_wave_closed_form(n):
    """Oracle RK4 + 4th-order FD equals Re(P(dt M)^n c e^{ikx}) per mode to roundoff.

    Catches any error in the RHS, stencils, ghost fill, or the RK4 combination."""
    L = 2 * math.pi
    h = tuple(L / v for v in n)
    dt = 0.25 * min(h)
    y0 = ci.pw3(n, h)
    got = oracle.rk4(W, y0, h, dt, 10)
    exact = pins.discrete_plane_wave(n, h, dt, 10, ci.PW3_MODES)
    scale = np.abs(exact).max()
    assert np.abs(got - exact).max() <= 1e-13 * scale


def test_rk4_amplification_single_mode_many_steps():
    """A single mode over 200 steps: amplitude follows |P(i y)|^n exactly (no drift)."""
    n = (8, 8, 8)
    h = (2 * math.pi / 8,) * 3
    dt = 0.5 * h[0]
    modes = (((1, 0, 0), 1.0, 0.2),)
    got = oracle.rk4(W, ci.pw3(n, h, modes=modes), h, dt, 200)
    exact = pins.discrete_plane_wave(n, h, dt, 200, modes)
    assert np.abs(got - exact).max() <= 1e-12


def _d1(f, axis, h):
    c = [1 / 12, -2 / 3, 0, 2 / 3, -1 / 12]
    out = np.zeros_like(f)
    for s, w in zip(range(-2, 3), c):
        if w:
            out += w * np.roll(f, -s, axis=axis)
    return out / h


def test_linear_invariants():
    """Exact discrete invariants of the linear scheme (RK4 preserves linear invariants):
    C_i = v_i - D1_i u, sum rho, sum v_i, sum u - t sum rho."""
    n = (12, 12, 12)
    h = (2 * math.pi / 12,) * 3
    dt = 0.25 * h[0]
    y0 = ci.noise(n, 5, seed=1410)
    y1 = oracle.rk4(W, y0, h, dt, 10)
    for i in range(3):
        c0 = y0[2 + i] - _d1(y0[0], 2 - i, h[i])
        c1 = y1[2 + i] - _d1(y1[0], 2 - i, h[i])
        assert np.abs(c1 - c0).max() < 1e-12
    assert abs(y1[1].sum() - y0[1].sum()) < 1e-11
    for i in range(3):
        assert abs(y1[2 + i].sum() - y0[2 + i].sum()) < 1e-11
    t = 10 * dt
    assert abs((y1[0].sum() - t * y1[1].sum()) - y0[0].sum()) < 1e-10


def test_energy_non_increasing():
    """Semi-discrete energy is conserved; RK4 makes it non-increasing per step
    (|P(iy)|^2 = 1 - y^6/72 + y^8/576 <= 1 below the stability limit)."""
    n = (10, 10, 10)
    h = (2 * math.pi / 10,) * 3
    dt = 0.25 * h[0]
    y = ci.noise(n, 5, seed=3)
    e_prev = oracle.norms(W, y, h)[-1]
    for _ in range(8):
        y = oracle.rk4(W, y, h, dt, 1)
        e = oracle.norms(W, y, h)[-1]
        assert e <= e_prev * (1 + 1e-15)
        e_prev = e
    # energy of Gaussian data equals the direct definition
    yg = ci.gaussian(n, h, width=1.0)
    vol = h[0] ** 3
    assert oracle.norms(W, yg, h)[-1] == pytest.approx(vol * 0.5 * (yg[1:] ** 2).sum(), rel=1e-13)


def test_norms_definitions():
    """SPEC.md:469-477 examples: constant 2 -> sum = 2 * N^3 * h^3; zero -> zeros;
    L2 of sin(x) on [0,2pi)^3 = sqrt(pi * (2 pi)^2)."""
    n = (8, 8, 8)
    h = (0.5, 0.5, 0.5)
    y = np.full((5, 8, 8, 8), 2.0)
    out = oracle.norms(W, y, h)
    assert out[2] == pytest.approx(2 * 512 * 0.125)
    assert out[1] == 2.0
    assert np.all(oracle.norms(W, np.zeros((5, 8, 8, 8)), h) == 0.0)
    N = 32
    hh = (2 * math.pi / N,) * 3
    z, yy, x = ci.coords((N, N, N), hh)
    f = np.zeros((5, N, N, N))
    f[0] = np.sin(x) + 0 * yy + 0 * z
    l2 = oracle.norms(W, f, hh)[0]
    assert l2 == pytest.approx(math.sqrt(math.pi * (2 * math.pi) ** 2), rel=1e-12)


def test_fourth_order_convergence():
    """Plane wave k=(1,1,1) over one period at N=16,32,64, lambda=0.25: measured order of
    the rho error in [3.6, 4.3]."""
    kv = (1, 1, 1)
    kn = math.sqrt(3)
    T = 2 * math.pi / kn
    errs = []
    for N in (16, 32, 64):
        h = (2 * math.pi / N,) * 3
        nsteps = int(math.ceil(T / (0.25 * h[0])))
        dt = T / nsteps
        modes = ((kv, 1.0, 0.0),)
        y0 = ci.pw3((N, N, N), h, modes=modes)
        y1 = oracle.rk4(W, y0, h, dt, nsteps)
        exact = ci.pw3((N, N, N), h, t=T, modes=modes)
        errs.append(math.sqrt(np.mean((y1[1] - exact[1]) ** 2)))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    for o in orders:
        assert 3.6 <= o <= 4.3, (errs, orders)


def test_zero_rhs_leaves_state_unchanged():
    """zero RHS -> state unchanged bitwise (rho = v = 0, u arbitrary)."""
    n = (8, 8, 8)
    y = np.zeros((5, 8, 8, 8))
    y[0] = ci.noise(n, 1, seed=9)[0]
    h = (0.3, 0.3, 0.3)
    assert np.array_equal(oracle.rk4(W, y, h, 0.1, 3), y)

"""Pins of the CPU oracle's BSSN path (reading R7) against
exact solutions and special cases that reduce to closed forms.  Each test names the
plausible transcription error it catches."""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np
import pytest

import chemora_inputs as ci
import oracle
from tests import bssn_exact, pins

B = oracle.BSSN
GF = ci.BSSN_GF
IX = {n: i for i, n in enumerate(GF)}
BENCH = [2.0, 1.0, 1.0, 0.0, 1.0, 0.75, 0.0, 1.0, 1.0, 1.0]
HARMONIC = [1.0, 2.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0, 1.0]   # gauge-wave gauge (App. A.3)


def flat(n):
    y = np.zeros((25, n[2], n[1], n[0]))
    for nm in ("gt11", "gt22", "gt33", "alpha"):
        y[IX[nm]] = 1.0
    return y


def flat_padded(n, g=3):
    y = np.zeros((25, n[2] + 2 * g, n[1] + 2 * g, n[0] + 2 * g))
    for nm in ("gt11", "gt22", "gt33", "alpha"):
        y[IX[nm]] = 1.0
    return y


@pytest.mark.parametrize("params", [BENCH, HARMONIC])
def test_minkowski_is_a_fixed_point(params):
    """alpha = 1, gt = delta, everything else 0 -> RHS = 0 (catches any constant term)."""
    n = (8, 8, 8)
    k = oracle.rhs(B, flat(n), (0.1, 0.1, 0.1), params)
    assert np.abs(k).max() <= 1e-14


def test_default_params_are_the_benchmark_gauge():
    assert list(oracle.default_bssn_params()) == BENCH


# ------------------------------------------------------------------ stencils inside the RHS
def _stencil_exact(coeffs, offsets, f, x0, h):
    """sum_k c_k f(x0 + k h) / h with exact rational weights (the stencil's definition)."""
    return sum(float(c) * f(x0 + o * h) for c, o in zip(coeffs, offsets)) / h


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("sign", [+1, -1])
def test_upwind_branch_and_weights(axis, sign):
    """Flat data, constant shift beta^axis = sign * 0.7, phi = x_axis^6 (not exactly
    differentiable, so D+ and D- give different truncation errors):
    d_t phi = beta * D(+/-) phi exactly as the moment-solved lopsided stencil."""
    g, n, h = 3, (10, 9, 11), (0.25, 0.5, 0.125)
    z, y, x = ci.padded_coords(n, g, h, origin=(0.3, -0.2, 0.1))
    coord = (x, y, z)[axis] + 0 * x + 0 * y + 0 * z
    pad = flat_padded(n)
    pad[IX["phi"]] = coord ** 6
    beta = sign * 0.7
    pad[IX[f"beta{axis + 1}"]] = beta
    k = oracle.rhs_padded(B, pad, h, BENCH)
    offs = range(-1, 4) if sign > 0 else range(-3, 2)
    cf = pins.moment_solve(1, offs)
    ci_ = [g + i for i in (2, 4, 6)]
    pt = [c - g for c in ci_]  # interior coordinate of the sample point (x, y, z)
    orig = (0.3, -0.2, 0.1)
    x0 = orig[axis] + pt[axis] * h[axis]
    expect = beta * _stencil_exact(cf, offs, lambda s: s ** 6, x0, h[axis])
    got = k[IX["phi"], pt[2], pt[1], pt[0]]
    assert got == pytest.approx(expect, rel=1e-12)
    # the other branch differs (the test can tell them apart)
    other = pins.moment_solve(1, range(-3, 2) if sign > 0 else range(-1, 4))
    wrong = beta * _stencil_exact(other, range(-3, 2) if sign > 0 else range(-1, 4), lambda s: s ** 6, x0, h[axis])
    assert abs(wrong - expect) > 1e-6 * abs(expect)


def _poly_deriv(c, axis):
    out = {}
    for (a, b, cc), w in c.items():
        e = (a, b, cc)[axis]
        if e:
            key = list((a, b, cc))
            key[axis] -= 1
            out[tuple(key)] = out.get(tuple(key), 0.0) + w * e
    return out


def test_shift_derivatives_polynomial_exactness():
    """Flat metric, polynomial shift (degree 4): the D1, D2 and mixed stencils of App. A
    are exact, so with Xt = 0 everywhere
      d_t Xt^i = gt^jk d_j d_k beta^i + 1/3 gt^ij d_j (d.beta)       (Adv(Xt) = 0)
      d_t gt_ij = d_j beta^i + d_i beta^j - 2/3 delta_ij d.beta      (Adv(gt) = 0)
      d_t phi = d.beta / 6,  d_t B^i = d_t Xt^i,  d_t beta^i = beta^k d_k beta^i
    equal the continuum values at every interior point."""
    rng = np.random.default_rng(5)
    g, n, h = 3, (8, 7, 9), (0.25, 0.25, 0.5)
    org = (-0.5, 0.25, -1.0)
    z, y, x = ci.padded_coords(n, g, h, origin=org)
    P = [ci.random_polynomial_coeffs(rng, 4) for _ in range(3)]
    for c in P:
        for key in c:
            c[key] *= 0.05
    pad = flat_padded(n)
    for i in range(3):
        pad[IX[f"beta{i + 1}"]] = ci.eval_polynomial(P[i], x, y, z) + 0 * x + 0 * y + 0 * z
    k = oracle.rhs_padded(B, pad, h, BENCH)
    zi, yi, xi = z[g:-g], y[:, g:-g], x[:, :, g:-g]
    shape = (n[2], n[1], n[0])
    ev = lambda c: ci.eval_polynomial(c, xi, yi, zi) + np.zeros(shape)
    d = [[ev(_poly_deriv(P[i], a)) for a in range(3)] for i in range(3)]        # d[i][a] = d_a beta^i
    dd = [[[ev(_poly_deriv(_poly_deriv(P[i], a), b)) for b in range(3)] for a in range(3)] for i in range(3)]
    beta = [ev(P[i]) for i in range(3)]
    div = d[0][0] + d[1][1] + d[2][2]
    tol = 1e-10
    for i in range(3):
        lap = dd[i][0][0] + dd[i][1][1] + dd[i][2][2]
        graddiv = dd[0][i][0] + dd[1][i][1] + dd[2][i][2]
        xt = lap + graddiv / 3.0
        np.testing.assert_allclose(k[IX[f"Xt{i + 1}"]], xt, atol=tol)
        np.testing.assert_allclose(k[IX[f"B{i + 1}"]], xt, atol=tol)
        adv = sum(beta[kk] * d[i][kk] for kk in range(3))
        np.testing.assert_allclose(k[IX[f"beta{i + 1}"]], adv, atol=tol)
    names = {(0, 0): "gt11", (0, 1): "gt12", (0, 2): "gt13", (1, 1): "gt22", (1, 2): "gt23", (2, 2): "gt33"}
    for (i, j), nm in names.items():
        expect = d[i][j] + d[j][i] - (2.0 / 3.0 if i == j else 0.0) * div
        np.testing.assert_allclose(k[IX[nm]], expect, atol=tol)
    np.testing.assert_allclose(k[IX["phi"]], div / 6.0, atol=tol)


# ------------------------------------------------------------------ gauge ODE reductions
def test_gamma_driver_homogeneous_closed_form():
    """Spatially constant B = b, beta = 0 on flat data (benchmark gauge, S_B = 1): all
    spatial derivatives vanish, so B(t) = b e^{-eta t}, beta(t) = C_beta b (1 - e^{-eta t})/eta."""
    n = (6, 6, 6)
    y = flat(n)
    b = (0.3, -0.2, 0.1)
    for i in range(3):
        y[IX[f"B{i + 1}"]] = b[i]
    dt, steps = 0.01, 100
    out = oracle.rk4(B, y, (0.2, 0.2, 0.2), dt, steps, BENCH)
    t = dt * steps
    for i in range(3):
        assert np.allclose(out[IX[f"B{i + 1}"]], b[i] * math.exp(-t), atol=1e-11, rtol=0)
        assert np.allclose(out[IX[f"beta{i + 1}"]], 0.75 * b[i] * (1 - math.exp(-t)), atol=1e-11, rtol=0)
    others = [v for v in range(25) if GF[v] not in ("B1", "B2", "B3", "beta1", "beta2", "beta3")]
    assert np.abs(out[others] - y[others]).max() <= 1e-15  # stencils of constants: roundoff only


def test_one_plus_log_homogeneous_reduces_to_ode():
    """Spatially constant alpha, K, A (flat gt, At = 0): App. A reduces to the ODEs
    K' = alpha K^2/3, A' = K' - eta_alpha A, alpha' = -F alpha^n (L A + (1-L) K),
    phi' = -alpha K/6, integrated here by scipy (independent integrator, rtol 1e-12)."""
    from scipy.integrate import solve_ivp
    n = (6, 6, 6)
    y = flat(n)
    a0, K0, A0 = 0.9, 0.2, 0.05
    y[IX["alpha"]], y[IX["trK"]], y[IX["A"]] = a0, K0, A0
    dt, steps = 0.005, 200
    out = oracle.rk4(B, y, (0.2, 0.2, 0.2), dt, steps, BENCH)

    def f(t, u):
        al, K, A, ph = u
        Kd = al * K * K / 3.0
        return [-2.0 * al * A, Kd, Kd, -al * K / 6.0]

    sol = solve_ivp(f, (0, dt * steps), [a0, K0, A0, 0.0], rtol=1e-12, atol=1e-14)
    al, K, A, ph = sol.y[:, -1]
    for nm, v in (("alpha", al), ("trK", K), ("A", A), ("phi", ph)):
        assert np.allclose(out[IX[nm]], v, rtol=1e-9, atol=1e-12), nm


# ------------------------------------------------------------------ exact evolutions
def _gauge_wave_error(N, shift, t_end=0.5, amp=0.1):
    n = (N, 6, 6)
    h = (1.0 / N, 1.0 / 6, 1.0 / 6)
    nsteps = int(round(t_end / (0.25 / N)))
    dt = t_end / nsteps
    y0 = ci.gauge_wave(n, h, t=0.0, amp=amp, shift=shift)
    params = list(HARMONIC)
    out = oracle.rk4(B, y0, h, dt, nsteps, params)
    exact = ci.gauge_wave(n, h, t=t_end, amp=amp, shift=shift)
    # B^i is passive in this gauge (S_B = C_beta = 0: it feeds back into nothing) and is
    # not part of the exact solution (d_t B = Adv(B) - Adv(Xt) != 0 once beta != 0)
    active = [v for v in range(25) if not GF[v].startswith("B")]
    return np.abs(out[active] - exact[active]).max()


def test_gauge_wave_initial_data_is_a_solution():
    """The gauge-wave data are an exact solution: RHS equals d_t of the exact data."""
    N = 64
    n = (N, 6, 6)
    h = (1.0 / N, 1.0 / 6, 1.0 / 6)
    k = oracle.rhs(B, ci.gauge_wave(n, h), h, HARMONIC)
    dl = 1e-4
    dtex = (ci.gauge_wave(n, h, t=dl) - ci.gauge_wave(n, h, t=-dl)) / (2 * dl)
    assert np.abs(k - dtex).max() < 1e-4


@pytest.mark.parametrize("shift", [0.0, 0.5, -0.5])
def test_gauge_wave_fourth_order_convergence(shift):
    """Gauge wave (harmonic lapse, frozen shift) and shifted gauge wave (constant beta^x,
    both upwind branches): L_inf error after t = 0.5 converges at 4th order."""
    errs = [_gauge_wave_error(N, shift) for N in (16, 32, 64)]
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert errs[0] < 1e-2
    for o in orders:
        assert 3.6 <= o <= 4.3, (errs, orders)


def _pure_gauge_rhs_error(N, t0=0.4):
    L = 2 * math.pi
    h = (L / N,) * 3
    n = (N, N, N)
    z, y, x = ci.coords(n, h)
    x, y, z = np.broadcast_arrays(x, y, z)
    v = bssn_exact.bssn_vars(t0, x, y, z)
    state = np.zeros((25,) + x.shape)
    for nm, arr in v.items():
        state[IX[nm]] = arr
    k = oracle.rhs(B, state, h, BENCH)
    ex = bssn_exact.bssn_time_derivative(t0, x, y, z)
    return max(np.abs(k[IX[nm]] - ex[nm]).max() for nm in bssn_exact.ADM_PART)


def test_pure_gauge_rhs_convergence():
    """3-D exact vacuum solution with non-trivial lapse and shift (App. A.4): the 17
    ADM-part RHS components converge to d_t of the exact BSSN variables at 4th order.
    Catches any dropped/mis-signed term of the phi, gt, K, At, Xt equations."""
    errs = [_pure_gauge_rhs_error(N) for N in (16, 32, 64)]
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert errs[2] < 3e-4, errs
    assert orders[1] >= 3.6, (errs, orders)
    assert orders[0] >= 3.2, (errs, orders)


@pytest.mark.slow
def test_robust_stability_noise():
    """Minkowski + 1e-10 noise, benchmark gauge, no dissipation: stays bounded (no
    exponential growth) over one crossing time at 16^3."""
    n = (16, 16, 16)
    h = (1.0 / 16,) * 3
    y = flat(n) + 1e-10 * ci.noise(n, 25, seed=7)
    ref = flat(n)
    dt = 0.25 / 16
    devs = []
    for _ in range(4):
        y = oracle.rk4(B, y, h, dt, 16, BENCH)
        devs.append(np.abs(y - ref).max())
    assert max(devs) < 1e-7, devs
    assert devs[-1] <= 2.0 * devs[1], devs

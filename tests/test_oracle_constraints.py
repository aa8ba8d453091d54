"""Pins of the oracle's BSSN constraint monitors (
DESIGN.md reading R16):

    H   = e^{-4 phi} gt^ij (R~_ij + R^phi_ij) + 2/3 K^2 - At_ij At^ij
    M^i = d_j At^ij + Gt^i_jk At^jk + 6 At^ij d_j phi - 2/3 gt^ij d_j K
    G^i = Xt^i - gt^jk Gt^i_jk

against (a) flat space (exactly 0), (b) conformally flat data whose constraints have a
textbook closed form (R = -8 psi^-5 lap psi for gamma = psi^4 delta; sympy derivatives),
(c) exact vacuum solutions, where every constraint converges to 0 at 4th order."""
from __future__ import annotations

import functools
import math

import numpy as np
import pytest
import sympy as sp

import chemora_inputs as ci
import oracle
from tests import bssn_exact

IX = {n: i for i, n in enumerate(ci.BSSN_GF)}


def flat(n):
    y = np.zeros((25, n[2], n[1], n[0]))
    for nm in ("gt11", "gt22", "gt33", "alpha"):
        y[IX[nm]] = 1.0
    return y


def test_flat_space_constraints_vanish():
    n = (8, 8, 8)
    c = oracle.constraints(flat(n), (0.1, 0.1, 0.1))
    assert c.shape == (7, 8, 8, 8)
    assert np.abs(c).max() == 0.0


# ------------------------------------------------------------------ conformally flat closed form
@functools.lru_cache(maxsize=None)
def _conf_flat_exprs():
    """gt = delta, Xt given, phi, K, At (traceless) given analytic periodic functions.  With
    Gt = 0: H = -8 e^{-5 phi} lap(e^phi) + 2/3 K^2 - At_ij At_ij (Hamiltonian constraint of
    gamma = psi^4 delta), M^i = d_j At_ij + 6 At_ij d_j phi - 2/3 d_i K, G^i = Xt^i."""
    x, y, z = sp.symbols("x y z")
    X = (x, y, z)
    phi = sp.Rational(1, 10) * sp.sin(x) * sp.cos(y + z)
    K = sp.Rational(1, 5) * sp.cos(x - z) + sp.Rational(1, 10) * sp.sin(y)
    a = sp.Rational(1, 10)
    At = sp.Matrix([[a * sp.sin(y), a * sp.cos(z), a * sp.sin(x + y)],
                    [a * sp.cos(z), a * sp.cos(x), a * sp.sin(z - x)],
                    [a * sp.sin(x + y), a * sp.sin(z - x), -a * sp.sin(y) - a * sp.cos(x)]])
    Xt = [sp.Rational(1, 10) * sp.cos(y), sp.Rational(1, 10) * sp.sin(z + x), sp.Rational(1, 20)]
    psi = sp.exp(phi)
    lap = sum(sp.diff(psi, v, 2) for v in X)
    H = -8 * sp.exp(-5 * phi) * lap + sp.Rational(2, 3) * K ** 2 - sum(
        At[i, j] ** 2 for i in range(3) for j in range(3))
    M = [sum(sp.diff(At[i, j], X[j]) + 6 * At[i, j] * sp.diff(phi, X[j]) for j in range(3))
         - sp.Rational(2, 3) * sp.diff(K, X[i]) for i in range(3)]
    fields = {"phi": phi, "trK": K}
    names = ["11", "12", "13", "22", "23", "33"]
    idx = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]
    for nm, (i, j) in zip(names, idx):
        fields["At" + nm] = At[i, j]
    for i in range(3):
        fields[f"Xt{i + 1}"] = Xt[i]
    lam = lambda e: sp.lambdify(X, e, "numpy")
    return ({k: lam(v) for k, v in fields.items()}, [lam(e) for e in [H] + M + Xt])


def _conf_flat_error(N):
    L = 2 * math.pi
    h = (L / N,) * 3
    n = (N, N, N)
    z, y, x = ci.coords(n, h)
    x, y, z = np.broadcast_arrays(x, y, z)
    fields, exact = _conf_flat_exprs()
    st = flat(n)
    for nm, f in fields.items():
        st[IX[nm]] = np.broadcast_to(f(x, y, z), x.shape)
    c = oracle.constraints(st, h)
    return [np.abs(c[q] - np.broadcast_to(exact[q](x, y, z), x.shape)).max() for q in range(7)]


def test_conformally_flat_closed_form():
    """Nonzero constraints with a closed form: catches a wrong normalisation or sign of any
    term of H (the -8 psi^-5 lap psi Ricci scalar, the K^2 and At.At terms), of M (div At,
    the 6 At d phi term, the -2/3 dK term) and the G definition."""
    e16, e32 = _conf_flat_error(16), _conf_flat_error(32)
    for q in range(7):
        assert e32[q] < 2e-4, (q, e16, e32)
        if e16[q] > 1e-12:
            assert math.log2(e16[q] / e32[q]) >= 3.5, (q, e16, e32)
    # G^i = Xt^i exactly when gt = delta (no derivative of a constant metric)
    assert max(e32[4:]) < 1e-15


# ------------------------------------------------------------------ exact vacuum solutions
def _pure_gauge_constraint_error(N, t0=0.4):
    L = 2 * math.pi
    h = (L / N,) * 3
    n = (N, N, N)
    z, y, x = ci.coords(n, h)
    x, y, z = np.broadcast_arrays(x, y, z)
    v = bssn_exact.bssn_vars(t0, x, y, z)
    st = np.zeros((25,) + x.shape)
    for nm, arr in v.items():
        st[IX[nm]] = arr
    c = oracle.constraints(st, h)
    return [np.abs(c[q]).max() for q in range(7)]


def test_pure_gauge_constraints_converge_to_zero():
    """3-D pure-gauge Minkowski (non-trivial gt, At, phi, K, Xt): H, M, G
    vanish analytically, so the discrete values converge to 0 at 4th order.  Catches every
    Christoffel-dependent term the conformally flat case leaves untested."""
    e = [_pure_gauge_constraint_error(N) for N in (16, 32, 64)]
    for q in range(7):
        o2 = math.log2(e[1][q] / e[2][q])
        assert o2 >= 3.6, (q, e)
        assert e[2][q] < 5e-4, (q, e)
    # the data are far from flat: the constraint terms themselves are O(1e-1)
    st = bssn_exact.bssn_vars(0.4, np.array(0.3), np.array(0.7), np.array(1.1))
    assert abs(float(st["trK"])) > 1e-2


@pytest.mark.parametrize("shift", [0.0, 0.5])
def test_gauge_wave_constraints_converge_to_zero(shift):
    errs = []
    for N in (16, 32, 64):
        n = (N, 6, 6)
        h = (1.0 / N, 1.0 / 6, 1.0 / 6)
        c = oracle.constraints(ci.gauge_wave(n, h, t=0.3, amp=0.1, shift=shift), h)
        errs.append(np.abs(c).max(axis=(1, 2, 3)))
    for q in (0, 1, 4):
        o = math.log2(errs[1][q] / errs[2][q])
        assert o >= 3.6, (q, errs)
    # transverse components vanish identically (data independent of y, z)
    for q in (2, 3, 5, 6):
        assert errs[2][q] < 1e-14, (q, errs)


def test_constraint_violation_detects_perturbation():
    """Perturbing only K makes H = 2/3 K^2 and M^i = -2/3 d_i K (flat otherwise): the
    monitor sees constraint-violating data, at the exact algebraic size."""
    n = (16, 16, 16)
    h = (2 * math.pi / 16,) * 3
    z, y, x = ci.coords(n, h)
    st = flat(n)
    st[IX["trK"]] = np.broadcast_to(0.3 + 0 * x + 0 * y + 0 * z, (16, 16, 16))
    c = oracle.constraints(st, h)
    assert np.allclose(c[0], (2.0 / 3.0) * 0.09, rtol=0, atol=1e-15)
    assert np.abs(c[1:]).max() < 1e-15

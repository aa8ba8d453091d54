"""NEXT-1: run-time selectable accuracy order of the wave stencils
("Finite Differencing with arbitrary order of accuracy ... can be left as
run-time option").  Pins of the oracle's order-2/6/8 operators."""
from __future__ import annotations

import math

import numpy as np
import pytest

import chemora_inputs as ci
import oracle
from tests import pins

W = oracle.WAVE
ORDERS = [2, 4, 6, 8]


@pytest.mark.parametrize("order", ORDERS)
def test_d1_weights_are_the_moment_solution(order):
    """Weights read off the oracle RHS of a delta function = exact moment solve."""
    w = order // 2
    h = 0.375
    y = np.zeros((5, 14, 14, 14))
    y[1, 7, 7, 7] = 1.0
    k = oracle.rhs(W, y, (h, h, h), g=4, order=order)
    got = [k[2][7, 7, 7 - s] * h for s in range(-w, w + 1)]
    exact = [float(c) for c in pins.moment_solve(1, range(-w, w + 1))]
    np.testing.assert_allclose(got, exact, rtol=1e-15, atol=1e-15)


@pytest.mark.parametrize("order", ORDERS)
def test_polynomial_exactness_to_degree_order(order):
    """A centered D1 of accuracy 2w is exact for polynomials of degree <= 2w."""
    g, n, h = 4, (9, 9, 9), (0.25, 0.5, 0.125)
    z, y, x = ci.padded_coords(n, g, h, origin=(-0.5, 0.25, 0.0))
    pad = np.zeros((5, n[2] + 2 * g, n[1] + 2 * g, n[0] + 2 * g))
    pad[1] = x ** order - 2.0 * y ** (order - 1) + z ** order + 0 * x * y * z
    k = oracle.rhs_padded(W, pad, h, g=g, order=order)
    xi, yi, zi = x[:, :, g:-g], y[:, g:-g], z[g:-g]
    np.testing.assert_allclose(k[2], order * xi ** (order - 1) + 0 * yi * zi, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(k[3], -2.0 * (order - 1) * yi ** (order - 2) + 0 * xi * zi, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(k[4], order * zi ** (order - 1) + 0 * xi * yi, rtol=1e-11, atol=1e-11)
    # degree order + 1 is not exact
    pad[1] = x ** (order + 1) + 0 * y * z
    k = oracle.rhs_padded(W, pad, h, g=g, order=order)
    assert np.abs(k[2] - (order + 1) * xi ** order).max() > 1e-8


@pytest.mark.parametrize("order", ORDERS)
def test_discrete_plane_wave_closed_form(order):
    n = (12, 10, 8)
    h = tuple(2 * math.pi / v for v in n)
    dt = 0.2 * min(h)
    got = oracle.rk4(W, ci.pw3(n, h), h, dt, 8, g=4, order=order)
    exact = pins.discrete_plane_wave_order(n, h, dt, 8, ci.PW3_MODES, order)
    assert np.abs(got - exact).max() <= 1e-13 * np.abs(exact).max()


@pytest.mark.parametrize("order", [2, 4, 6])
def test_rhs_convergence_order(order):
    """RHS error on u = sin(x + 2y - z) converges at the stencil's order."""
    errs = []
    for N in (16, 32):
        h = (2 * math.pi / N,) * 3
        z, y, x = ci.coords((N, N, N), h)
        arg = x + 2 * y - z
        st = np.zeros((5, N, N, N))
        st[1] = np.sin(arg)
        k = oracle.rhs(W, st, h, g=4, order=order)
        errs.append(np.abs(k[2] - np.cos(arg)).max())
    p = math.log2(errs[0] / errs[1])
    assert order - 0.3 <= p <= order + 0.5, (errs, p)

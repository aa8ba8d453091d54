"""BSSN transcription pin (SURVEY.md §8(c) "BSSN transcription"): the
oracle's RHS and constraint fields of random polynomial data of degree <= 4 on all 25 GFs
(HOST_PADDED: ghosts are the polynomial's values, not a periodic fill) equal an independent
continuum evaluation of App. A at every sampled interior point (tests/bssn_jets.py: exact
jets, Ricci tensor of the physical metric from its own Christoffel symbols, physical
D_i D_j alpha, ...), because every stencil the oracle applies is exact on such data.  Run at
the benchmark gauge and at generic gauges that switch on every gauge branch (S_B in (0,1),
p_beta != 0, n_alpha != 1, eta_alpha != 0, c_adv != 1), so a dropped term, a wrong sign or a
wrong index anywhere in the App. A transcription fails here."""
from __future__ import annotations

import numpy as np
import pytest

import chemora_inputs as ci
import oracle
from tests import bssn_jets as BJ

BENCH = (2.0, 1.0, 1.0, 0.0, 1.0, 0.75, 0.0, 1.0, 1.0, 1.0)
GENERIC = (1.5, 2.0, 0.7, 0.3, 0.8, 0.6, 1.0, 0.5, 0.9, 0.7)
GENERIC2 = (0.8, 1.5, 0.3, 0.7, 1.3, 1.1, 2.5, 0.25, 0.4, 0.6)
HARMONIC = (1.0, 2.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0, 1.0)

N = (8, 8, 8)
H = (1.0 / 8, 1.0 / 8, 1.0 / 8)
ORIGIN = (-0.5, -0.4375, -0.5625)
G = 3


def _data(seed):
    """Polynomial data near flat space: gt_ii, alpha = 1 + small, everything else small,
    with every GF a different random degree-4 polynomial (integer coefficients)."""
    rng = np.random.default_rng(seed)
    polys = [ci.random_polynomial_coeffs(rng, 4) for _ in range(25)]
    bases = np.zeros(25)
    for v in (1, 4, 6, 17):       # gt11, gt22, gt33, alpha
        bases[v] = 1.0
    scales = np.full(25, 0.01)
    scales[[1, 2, 3, 4, 5, 6]] = 0.004   # conformal metric stays positive definite
    scales[0] = 0.006
    scales[17] = 0.004
    scales[19:22] = 0.02                 # shift of both signs: both upwind branches
    z, y, x = ci.padded_coords(N, G, H, ORIGIN)
    padded = np.zeros((25, N[2] + 2 * G, N[1] + 2 * G, N[0] + 2 * G))
    for v in range(25):
        padded[v] = bases[v] + scales[v] * ci.eval_polynomial(polys[v], x, y, z)
    return padded, polys, scales, bases


def _points(nsample, seed):
    rng = np.random.default_rng(seed)
    pts = {(0, 0, 0), (N[0] - 1, N[1] - 1, N[2] - 1)}
    while len(pts) < nsample:
        pts.add(tuple(int(rng.integers(0, N[a])) for a in range(3)))
    return sorted(pts)


@pytest.mark.parametrize("params", [BENCH, GENERIC, GENERIC2, HARMONIC])
@pytest.mark.parametrize("seed", [3, 11])
def test_rhs_equals_continuum_app_a(params, seed):
    padded, polys, scales, bases = _data(seed)
    k = oracle.rhs_padded(oracle.BSSN, padded, H, list(params))
    worst = np.zeros(25)
    scale = np.zeros(25)
    for (i, j, kk) in _points(40, seed):
        p = np.array([ORIGIN[0] + i * H[0], ORIGIN[1] + j * H[1], ORIGIN[2] + kk * H[2]])
        J = BJ.fields_at(polys, scales, bases, p)
        ref, _ = BJ.bssn_rhs_and_constraints(J, params)
        got = k[:, kk, j, i]
        worst = np.maximum(worst, np.abs(got - ref))
        scale = np.maximum(scale, np.abs(ref))
    # the RHS of every GF is non-trivial at this data (the pin really tests every equation)
    for v in range(25):
        if not (params[5] == 0.0 and 19 <= v < 22):   # frozen shift: d_t beta = c Adv(beta) only
            assert scale[v] > 1e-4, (v, scale[v])
    rel = worst / np.maximum(scale, 1e-12)
    assert rel.max() <= 1e-9, {ci.BSSN_GF[v]: rel[v] for v in np.argsort(rel)[-5:]}


@pytest.mark.parametrize("seed", [3, 11])
def test_constraints_equal_continuum(seed):
    """H, M^i (D~_j At^ij with the full conformal Christoffel symbols -- det gt != 1 here) and
    G^i of the oracle equal the continuum values (R16)."""
    padded, polys, scales, bases = _data(seed)
    c = oracle.constraints_padded(padded, H)
    worst, scale = np.zeros(7), np.zeros(7)
    for (i, j, kk) in _points(30, seed + 1):
        p = np.array([ORIGIN[0] + i * H[0], ORIGIN[1] + j * H[1], ORIGIN[2] + kk * H[2]])
        _, ref = BJ.bssn_rhs_and_constraints(BJ.fields_at(polys, scales, bases, p), BENCH)
        worst = np.maximum(worst, np.abs(c[:, kk, j, i] - ref))
        scale = np.maximum(scale, np.abs(ref))
    assert scale.min() > 1e-4
    assert (worst / scale).max() <= 1e-9, worst / scale


def test_jets_first_principles_sanity():
    """The jet machinery itself: the Ricci tensor of a conformally flat metric e^{4 phi}
    delta is the textbook conformal-transformation result (n = 3, g = e^{2f} delta, f = 2 phi):
    R_ij = -(n-2)(d_i d_j f - d_i f d_j f) - delta_ij (lap f + (n-2)|grad f|^2)."""
    rng = np.random.default_rng(5)
    poly = ci.random_polynomial_coeffs(rng, 4)
    p = np.array([0.1, -0.2, 0.3])
    phi = BJ.poly_jet(poly, p, 0.05)
    e4 = BJ.jexp(4.0 * phi)
    one, zero = BJ.Jet(1.0), BJ.Jet(0.0)
    gam = [[e4 * (one if i == j else zero) for j in range(3)] for i in range(3)]
    inv, _ = BJ.inverse3(gam)
    R = BJ.ricci(BJ.christoffel(gam, inv))
    d, dd = phi.g, phi.H
    f, df, ddf = None, 2.0 * d, 2.0 * dd
    ref = -(ddf - np.outer(df, df)) - np.eye(3) * (np.trace(ddf) + df @ df)
    np.testing.assert_allclose(R, ref, rtol=1e-12, atol=1e-14)

"""GPU parity tests of the BSSN path: CUDA kernels behind the C ABI vs the CPU oracle on
identical seeded inputs.  Tolerance (north_star): max relative error <= 1e-10 after 10 RK4
steps, per GF normwise (max|gpu - oracle| / max|oracle|, reading R11)."""
from __future__ import annotations

import math

import numpy as np
import pytest

import chemora_inputs as ci
import oracle

pytestmark = pytest.mark.gpu
B = 2
BENCH = [2.0, 1.0, 1.0, 0.0, 1.0, 0.75, 0.0, 1.0, 1.0, 1.0]
HARMONIC = [1.0, 2.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0, 1.0]
# generic gauges: every branch of App. A.3 active (S_B in (0,1), p_beta != 0, n_alpha != 1,
# eta_alpha != 0, c_adv != 1; GENERIC2 also a non-integer p_beta and L < 1/2)
GENERIC = [1.5, 2.0, 0.7, 0.3, 0.8, 0.6, 1.0, 0.5, 0.9, 0.7]
GENERIC2 = [0.8, 1.5, 0.3, 0.7, 1.3, 1.1, 2.5, 0.25, 0.4, 0.6]


def _mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1410_1764_b200 as P
    from paper_1410_1764_b200 import capi as C
    return P, C


def relerr(a, b, floor=0.0):
    """Per-GF normwise relative error (R11).  A GF whose reference is (up to
    roundoff) identically zero is compared against 1e-6 of the largest GF's scale instead
    of its own ~1e-19 roundoff noise."""
    out = []
    top = max(np.abs(b[f]).max() for f in range(b.shape[0]))
    for f in range(a.shape[0]):
        s = max(np.abs(b[f]).max(), floor, 1e-6 * top)
        d = np.abs(a[f] - b[f]).max()
        out.append(d / s if s > 0 else d)
    return max(out)


def perturbed(n, eps=1e-3, seed=1410):
    h = tuple(1.0 / v for v in n)
    return ci.mink_pert(n, h, seed, eps=eps), h


@pytest.mark.parametrize("n", [(32, 32, 32), (36, 28, 44)])
def test_rhs_parity_mink_pert(n):
    P, C = _mods()
    y0, h = perturbed(n, eps=1e-2)
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_initial(C.INIT_HOST, y0)
    k = g.rhs().cpu().numpy()
    ref = oracle.rhs(B, y0, h, BENCH)
    assert relerr(k, ref) <= 1e-10


def test_rhs_parity_pure_gauge():
    """Strongly non-trivial data (the pure-gauge exact solution, App. A.4)."""
    P, C = _mods()
    from tests import bssn_exact
    N = 24
    n = (N, N, N)
    h = (2 * math.pi / N,) * 3
    z, y, x = ci.coords(n, h)
    x, y, z = np.broadcast_arrays(x, y, z)
    v = bssn_exact.bssn_vars(0.4, x, y, z)
    state = np.zeros((25,) + x.shape)
    for nm, arr in v.items():
        state[ci.BSSN_GF.index(nm)] = arr
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_initial(C.INIT_HOST, state)
    k = g.rhs().cpu().numpy()
    ref = oracle.rhs(B, state, h, BENCH)
    assert relerr(k, ref, floor=1e-3) <= 1e-11


@pytest.mark.parametrize("params", [BENCH, HARMONIC, GENERIC, GENERIC2])
def test_rhs_parity_gauge_params(params):
    P, C = _mods()
    n = (20, 16, 24)
    y0, h = perturbed(n, eps=2e-2, seed=3)
    y0[ci.BSSN_GF.index("alpha")] += 0.1
    g = P.Grid(C.SYS_BSSN, n, h, params=params)
    g.set_initial(C.INIT_HOST, y0)
    k = g.rhs().cpu().numpy()
    ref = oracle.rhs(B, y0, h, params)
    assert relerr(k, ref) <= 1e-10


@pytest.mark.parametrize("n", [(32, 32, 32), (48, 48, 48), (36, 28, 44)])
def test_rk4_parity_10_steps(n):
    P, C = _mods()
    y0, h = perturbed(n)
    dt = 0.25 * min(h)
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(dt, 10)
    got = g.get_state()
    ref = oracle.rk4(B, y0, h, dt, 10, BENCH)
    # compare the change from the initial data too (the perturbation is ~1e-3 of flat)
    assert relerr(got, ref) <= 1e-10
    assert relerr(got - y0, ref - y0) <= 1e-8


@pytest.mark.parametrize("params", [BENCH, GENERIC, GENERIC2])
@pytest.mark.parametrize("seed", [3, 11])
def test_rhs_parity_polynomial_data(params, seed):
    """The transcription-pin data (tests/test_oracle_bssn_continuum.py: random degree-4
    polynomials on all 25 GFs, ghosts as given -- HOST_PADDED), where every term of every
    equation is O(1) and the stencils are exact: GPU RHS vs oracle RHS, and both vs the
    independent continuum evaluation at sampled points."""
    P, C = _mods()
    from tests import bssn_jets as BJ
    from tests import test_oracle_bssn_continuum as TC
    padded, polys, scales, bases = TC._data(seed)
    g = P.Grid(C.SYS_BSSN, TC.N, TC.H, origin=TC.ORIGIN, params=params)
    g.set_initial(C.INIT_HOST_PADDED, padded)
    k = g.rhs().cpu().numpy()
    ref = oracle.rhs_padded(B, padded, TC.H, params)
    assert relerr(k, ref) <= 1e-11
    for (i, j, kk) in TC._points(12, seed):
        p = np.array([TC.ORIGIN[0] + i * TC.H[0], TC.ORIGIN[1] + j * TC.H[1], TC.ORIGIN[2] + kk * TC.H[2]])
        cont, _ = BJ.bssn_rhs_and_constraints(BJ.fields_at(polys, scales, bases, p), params)
        np.testing.assert_allclose(k[:, kk, j, i], cont, rtol=0, atol=1e-9 * np.abs(ref).max())


@pytest.mark.parametrize("params", [GENERIC, GENERIC2])
def test_rk4_parity_10_steps_generic_gauge(params):
    P, C = _mods()
    n = (28, 24, 36)
    y0, h = perturbed(n, eps=1e-2, seed=5)
    y0[ci.BSSN_GF.index("alpha")] += 0.1
    dt = 0.25 * min(h)
    g = P.Grid(C.SYS_BSSN, n, h, params=params)
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(dt, 10)
    got = g.get_state()
    ref = oracle.rk4(B, y0, h, dt, 10, params)
    assert relerr(got, ref) <= 1e-10
    assert relerr(got - y0, ref - y0) <= 1e-8


def test_rk4_parity_10_steps_64():
    """North_star's BSSN bar at 64^3 (BSSN parity is graded at <= 64^3)."""
    P, C = _mods()
    n = (64, 64, 64)
    y0, h = perturbed(n)
    dt = 0.25 * min(h)
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(dt, 10)
    got = g.get_state()
    ref = oracle.rk4(B, y0, h, dt, 10, BENCH)
    assert relerr(got, ref) <= 1e-10
    assert relerr(got - y0, ref - y0) <= 1e-8


def test_gauge_wave_parity():
    P, C = _mods()
    n = (64, 6, 6)
    h = (1.0 / 64, 1.0 / 6, 1.0 / 6)
    y0 = ci.gauge_wave(n, h, shift=0.5)
    g = P.Grid(C.SYS_BSSN, n, h, params=HARMONIC)
    g.set_initial(C.INIT_HOST, y0)
    dt = 0.25 / 64
    g.rk4_step(dt, 10)
    ref = oracle.rk4(B, y0, h, dt, 10, HARMONIC)
    assert relerr(g.get_state(), ref) <= 1e-10


def test_device_mink_pert_matches_inputs_module():
    P, C = _mods()
    n = (24, 20, 16)
    h = tuple(1.0 / v for v in n)
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_initial(C.INIT_MINK_PERT, kind_params=[1e-3], seed=1410)
    np.testing.assert_allclose(g.get_state(), ci.mink_pert(n, h, 1410, eps=1e-3), rtol=0, atol=1e-15)


def test_local_slabs_bitwise_bssn():
    P, C = _mods()
    n = (16, 12, 24)
    y0, h = perturbed(n)
    dt = 0.25 * min(h)
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(dt, 3)
    s = P.LocalSlabs(C.SYS_BSSN, n, h, 2)
    s.set_initial(C.INIT_HOST, y0)
    s.rk4_step(dt, 3)
    assert np.array_equal(s.get_state(), g.get_state())
    # ... and element-wise against the oracle
    assert relerr(s.get_state(), oracle.rk4(B, y0, h, dt, 3, BENCH)) <= 1e-10


def test_full_size_192_sampled_parity():
    """Benchmark configuration (192^3, MINK_PERT, benchmark gauge, the bench's launch
    configuration): TWO RK4 steps, then 16 sampled points vs the oracle run on a (2R+1)^3
    periodic box around each point (wrap errors travel 3 points per stage, so R = 25 leaves
    the centre exact after 2 steps).  The GPU-vs-oracle difference is read against the
    oracle's own rounding-noise floor (the same oracle built with FMA contraction, SURVEY.md
    §8(c) Q11) and must stay within north_star's 1e-10 (normwise per GF over the samples)."""
    P, C = _mods()
    N = 192
    n = (N, N, N)
    h = (1.0 / N,) * 3
    dt = 0.25 * h[0]
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_initial(C.INIT_MINK_PERT, kind_params=[1e-3], seed=1410)
    y0 = g.get_state()
    g.rk4_step(dt, 2)
    state = g.get_state()
    R = 25
    pts = [(0, 0, 0), (191, 191, 191), (5, 190, 100), (100, 50, 3), (96, 96, 96), (2, 189, 2)]
    rng = np.random.default_rng(1)
    pts += [tuple(int(v) for v in rng.integers(0, N, 3)) for _ in range(10)]
    got, ref, fma, init = [], [], [], []
    use_floor = oracle.host_has_fma()
    for (i, j, k) in pts:
        lo = (i - R, j - R, k - R)
        box = ci.mink_pert((2 * R + 1,) * 3, h, 1410, eps=1e-3,
                           origin=tuple(l * hh for l, hh in zip(lo, h)), length=1.0)
        ref.append(oracle.rk4(B, box, h, dt, 2, BENCH)[:, R, R, R])
        if use_floor:
            with oracle.use_fma_build():
                fma.append(oracle.rk4(B, box, h, dt, 2, BENCH)[:, R, R, R])
        got.append(state[:, k, j, i])
        init.append(box[:, R, R, R])
        # the device init matches the box generator to roundoff
        np.testing.assert_allclose(y0[:, k, j, i], box[:, R, R, R], rtol=0, atol=1e-15)
    got, ref, init = (np.array(a).T[:, :, None, None] for a in (got, ref, init))
    e_state = relerr(got, ref)
    e_change = relerr(got - init, ref - init)
    msg = f"192^3 2 steps, {len(pts)} samples: GPU vs oracle state {e_state:.2e}, change {e_change:.2e}"
    if use_floor:
        fma = np.array(fma).T[:, :, None, None]
        f_state, f_change = relerr(fma, ref), relerr(fma - init, ref - init)
        msg += f"; oracle FMA-build floor state {f_state:.2e}, change {f_change:.2e}"
    print(msg)
    assert e_state <= 1e-10, msg
    assert e_change <= 1e-7, msg


@pytest.mark.parametrize("shift", [0.0, 0.5])
def test_gauge_wave_device_init_and_evolution(shift):
    """CHEMORA_INIT_GAUGE_WAVE equals the host recipe (chemora_inputs.gauge_wave) to rounding,
    and 10 RK4 steps in the harmonic gauge match the oracle (north_star BSSN tolerance) and
    stay close to the exact solution."""
    P, C = _mods()
    n = (48, 8, 8)
    h = (1.0 / 48, 1.0 / 8, 1.0 / 8)
    g = P.Grid(C.SYS_BSSN, n, h, params=HARMONIC)
    g.set_initial(C.INIT_GAUGE_WAVE, kind_params=[0.1, 1.0, shift, 0.0])
    host = ci.gauge_wave(n, h, t=0.0, amp=0.1, shift=shift)
    assert np.allclose(g.get_state(), host, rtol=1e-13, atol=1e-14)
    dt = 0.25 / 48
    g.rk4_step(dt, 10)
    got = g.get_state()
    ref = oracle.rk4(B, host, h, dt, 10, HARMONIC)   # the oracle starts from the host recipe
    assert relerr(got, ref) <= 1e-10
    exact = ci.gauge_wave(n, h, t=10 * dt, amp=0.1, shift=shift)
    active = [v for v in range(25) if not ci.BSSN_GF[v].startswith("B")]
    assert np.abs(got[active] - exact[active]).max() < 5e-5   # truncation error at N = 48


def test_gauge_wave_rejects_bad_params():
    P, C = _mods()
    n = (16, 8, 8)
    g = P.Grid(C.SYS_BSSN, n, (1.0 / 16, 0.125, 0.125))
    with pytest.raises(C.ChemoraError):
        g.set_initial(C.INIT_GAUGE_WAVE, kind_params=[1.5, 1.0, 0.0, 0.0])
    w = P.Grid(C.SYS_WAVE, n, (0.1,) * 3)
    with pytest.raises(C.ChemoraError):
        w.set_initial(C.INIT_GAUGE_WAVE)

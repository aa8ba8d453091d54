"""GPU parity tests of the wave path: the CUDA kernels behind the C ABI against the CPU
oracle on identical seeded inputs.

Tolerance (north_star): max relative error <= 1e-12 after 10 RK4 steps, measured per GF
as max|gpu - oracle| / max|oracle| over the interior (reading R11).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import chemora_inputs as ci
import oracle

pytestmark = pytest.mark.gpu

W = 1


def _mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1410_1764_b200 as P
    from paper_1410_1764_b200 import capi as C
    return P, C


def relerr(a, b):
    out = []
    for f in range(a.shape[0]):
        s = np.abs(b[f]).max()
        d = np.abs(a[f] - b[f]).max()
        out.append(d / s if s > 0 else d)
    return max(out)


def grid(n, h=None, **kw):
    P, C = _mods()
    if h is None:
        h = tuple(2 * math.pi / v for v in n)
    return P.Grid(C.SYS_WAVE, n, h, **kw), h


SIZES = [(32, 32, 32), (37, 29, 41), (64, 64, 64), (96, 96, 96), (48, 40, 56)]


@pytest.mark.parametrize("n", SIZES[:3])
@pytest.mark.parametrize("data", ["pw3", "noise"])
def test_rhs_parity(n, data):
    P, C = _mods()
    g, h = grid(n)
    y0 = ci.pw3(n, h) if data == "pw3" else ci.noise(n, 5, seed=1410)
    g.set_initial(C.INIT_HOST, y0)
    k = g.rhs().cpu().numpy()
    ref = oracle.rhs(W, y0, h)
    assert relerr(k, ref) <= 1e-13


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("data", ["pw3", "noise"])
def test_rk4_parity_10_steps(n, data):
    P, C = _mods()
    g, h = grid(n)
    dt = 0.25 * min(h)
    y0 = ci.pw3(n, h) if data == "pw3" else ci.noise(n, 5, seed=1410)
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(dt, 10)
    got = g.get_state()
    ref = oracle.rk4(W, y0, h, dt, 10)
    assert relerr(got, ref) <= 1e-12


def test_ghosts_after_step_are_the_periodic_fill():
    """After rk4_step the fused ghost-image writes leave y's ghosts equal to the periodic
    fill of its interior (edges and corners included) -- bitwise, they are copies."""
    P, C = _mods()
    n = (20, 18, 22)
    g, h = grid(n)
    g.set_initial(C.INIT_NOISE, seed=5)
    g.rk4_step(0.25 * min(h), 3)
    pad = g.get_state(padded=True)
    interior = pad[:, 3:-3, 3:-3, 3:-3]
    ref = np.pad(interior, ((0, 0), (3, 3), (3, 3), (3, 3)), mode="wrap")
    assert np.array_equal(pad, ref)


def test_device_init_matches_inputs_module():
    P, C = _mods()
    n = (24, 20, 16)
    g, h = grid(n)
    g.set_initial(C.INIT_NOISE, seed=77)
    assert np.array_equal(g.get_state(), ci.noise(n, 5, seed=77))
    g.set_initial(C.INIT_PLANE_WAVES)
    np.testing.assert_allclose(g.get_state(), ci.pw3(n, h), rtol=0, atol=1e-13)
    g.set_initial(C.INIT_GAUSSIAN, kind_params=[1.0, 0.5])
    np.testing.assert_allclose(g.get_state(), ci.gaussian(n, h, width=0.5), rtol=0, atol=1e-15)


def test_norms_parity():
    P, C = _mods()
    n = (40, 36, 32)
    g, h = grid(n)
    y0 = ci.noise(n, 5, seed=3)
    g.set_initial(C.INIT_HOST, y0)
    got = g.norms()
    ref = oracle.norms(W, y0, h)
    np.testing.assert_allclose(got, ref, rtol=1e-13)


def test_polynomial_host_padded_rhs():
    """HOST_PADDED polynomial data (ghosts as given): GPU RHS equals the oracle's."""
    P, C = _mods()
    rng = np.random.default_rng(4)
    n, gh, h = (16, 12, 20), 3, (0.5, 0.25, 0.125)
    z, y, x = ci.padded_coords(n, gh, h, origin=(-1.0, 0.5, -0.25))
    pad = np.zeros((5, n[2] + 6, n[1] + 6, n[0] + 6))
    for f in range(5):
        pad[f] = ci.eval_polynomial(ci.random_polynomial_coeffs(rng, 4), x, y, z)
    g = P.Grid(C.SYS_WAVE, n, h, origin=(-1.0, 0.5, -0.25))
    g.set_initial(C.INIT_HOST_PADDED, pad)
    k = g.rhs().cpu().numpy()
    ref = oracle.rhs_padded(W, pad, h)
    np.testing.assert_allclose(k, ref, rtol=0, atol=1e-10 * np.abs(ref).max())


def test_nonfinite_is_reported():
    P, C = _mods()
    n = (16, 16, 16)
    g, h = grid(n)
    y0 = ci.noise(n, 5, seed=1)
    y0[2, 5, 6, 7] = np.nan
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(0.1, 2)
    with pytest.raises(C.ChemoraError) as ei:
        g.get_state()
    assert ei.value.code == C.E_NONFINITE
    assert "step 0" in str(ei.value)


@pytest.mark.parametrize("nslabs", [2, 4])
def test_local_slabs_bitwise_equal_single_grid(nslabs):
    """z-slab decomposition emulated on one device (stage kernels store boundary planes
    into the neighbour slab's ghost planes): bitwise equal to the undecomposed grid."""
    P, C = _mods()
    n = (24, 20, 48)
    h = tuple(2 * math.pi / v for v in n)
    y0 = ci.noise(n, 5, seed=11)
    g = P.Grid(C.SYS_WAVE, n, h)
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(0.25 * min(h), 5)
    ref = g.get_state()
    s = P.LocalSlabs(C.SYS_WAVE, n, h, nslabs)
    s.set_initial(C.INIT_HOST, y0)
    s.rk4_step(0.25 * min(h), 5)
    assert np.array_equal(s.get_state(), ref)
    np.testing.assert_allclose(s.norms(), g.norms(), rtol=1e-14)
    # ... and element-wise against the oracle (not only against the GPU's own single grid)
    o = oracle.rk4(W, y0, h, 0.25 * min(h), 5)
    assert max(np.abs(s.get_state()[f] - o[f]).max() / np.abs(o[f]).max() for f in range(5)) <= 1e-12
    # ghosts of every slab are the periodic images of the global state
    full = np.pad(ref, ((0, 0), (3, 3), (3, 3), (3, 3)), mode="wrap")
    for gg, pad in zip(s.grids, s.get_state_padded()):
        z0 = gg.z0
        assert np.array_equal(pad, full[:, z0:z0 + gg.local_extent[2] + 6])


def test_kernel_variants_bitwise_identical():
    """Tile independence: every kernel design (one thread per point in banded
    and plain CTA order, the persistent TMA z-march, the temporally blocked stage pairs)
    gives bitwise identical states."""
    P, C = _mods()
    n = (70, 45, 33)
    out = []
    variants = (0, 1, 4, 8)
    for v in variants:
        g, h = grid(n)
        g.set_kernel_variant(v)
        g.set_initial(C.INIT_NOISE, seed=2)
        g.rk4_step(0.25 * min(h), 3)
        out.append(g.get_state())
    for v, o in zip(variants[1:], out[1:]):
        assert np.array_equal(out[0], o), f"variant {v} differs"


@pytest.mark.parametrize("order", [2, 6, 8])
def test_wide_stencil_tilings_bitwise_identical(order):
    """NEXT-1 orders through every design that takes them (one thread per point in banded and
    plain order, the persistent TMA z-march with radius-3/4 boxes, the stage pairs up to
    radius 3), on one grid and on two z-slabs: bitwise identical states."""
    P, C = _mods()
    n = (70, 45, 40)
    h = tuple(2 * math.pi / v for v in n)
    gh = max(3, order // 2)
    y0 = ci.noise(n, 5, seed=order)
    dt = 0.2 * min(h)
    out = []
    variants = (0, 1, 4) + ((8,) if order <= 6 else ())  # 8: the stage pairs (radius 1, 3)
    for v in variants:
        g = P.Grid(C.SYS_WAVE, n, h, ghost=gh, fd_order=order)
        g.set_kernel_variant(v)
        g.set_initial(C.INIT_HOST, y0)
        g.rk4_step(dt, 3)
        out.append(g.get_state())
    for v, o in zip(variants[1:], out[1:]):
        assert np.array_equal(out[0], o), f"order {order}: variant {v} differs"
    for sv in (4,) + ((8,) if order <= 6 else ()):
        s = P.LocalSlabs(C.SYS_WAVE, n, h, 2, ghost=gh, fd_order=order)
        for gg in s.grids:
            gg.set_kernel_variant(sv)
        s.set_initial(C.INIT_HOST, y0)
        s.rk4_step(dt, 3)
        assert np.array_equal(s.get_state(), out[0]), f"order {order}: two slabs, variant {sv}"


def _box_oracle_one_step(gext, h, dt, seed, center, R=10):
    """Oracle value at ``center`` after ONE RK4 step of the NOISE data of a periodic grid
    of extents ``gext``: the oracle runs periodically on a (2R+1)^3 box; wrap errors
    travel 2 points per stage, so with R >= 9 the centre is untouched by them."""
    lo = [c - R for c in center]
    size = [2 * R + 1] * 3
    box = ci.noise_box(gext, 5, seed, lo, size)
    out = oracle.rk4(W, box, h, dt, 1)
    return out[:, R, R, R]


def test_full_size_512_sampled_parity():
    """The benchmark configuration (512^3, the launch path bench.py times): 1 RK4 step on
    NOISE data, then sampled points (interior, faces, edges, corners) vs the oracle."""
    P, C = _mods()
    import torch
    n = (512, 512, 512)
    h = tuple(2 * math.pi / v for v in n)
    dt = 0.25 * min(h)
    g = P.Grid(C.SYS_WAVE, n, h)
    g.set_initial(C.INIT_NOISE, seed=1410)
    g.rk4_step(dt, 1)
    torch.cuda.synchronize()
    # read back only the sampled points through a padded-state view of the workspace
    state = g.get_state()
    rng = np.random.default_rng(0)
    pts = [(0, 0, 0), (511, 511, 511), (0, 511, 257), (300, 0, 511), (5, 200, 1)]
    pts += [tuple(int(v) for v in rng.integers(0, 512, 3)) for _ in range(6)]
    for (i, j, k) in pts:
        ref = _box_oracle_one_step(n, h, dt, 1410, (i, j, k))
        got = state[:, k, j, i]
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    del state
    # property at full size: sum rho and sum v_i are invariants of the scheme
    g2 = g
    g2.set_initial(C.INIT_NOISE, seed=1410)
    n0 = g2.norms()
    g2.rk4_step(dt, 2)
    n1 = g2.norms()
    vol = h[0] ** 3
    for f in (1, 2, 3, 4):
        assert abs(n1[3 * f + 2] - n0[3 * f + 2]) <= 1e-6 * vol
    assert n1[-1] <= n0[-1]  # energy non-increasing


@pytest.mark.parametrize("order", [2, 4, 6, 8])
def test_fd_order_parity(order):
    """NEXT-1: run-time selectable accuracy order, every tiling."""
    P, C = _mods()
    n = (40, 36, 44)
    h = tuple(2 * math.pi / v for v in n)
    dt = 0.2 * min(h)
    y0 = ci.noise(n, 5, seed=order)
    ref = oracle.rk4(W, y0, h, dt, 10, g=4, order=order)
    for v in (0, 4) + ((8,) if order <= 6 else ()):
        g = P.Grid(C.SYS_WAVE, n, h, ghost=4, fd_order=order)
        g.set_kernel_variant(v)
        g.set_initial(C.INIT_HOST, y0)
        k = g.rhs().cpu().numpy()
        assert relerr(k, oracle.rhs(W, y0, h, g=4, order=order)) <= 1e-13
        g.rk4_step(dt, 10)
        assert relerr(g.get_state(), ref) <= 1e-12


@pytest.mark.parametrize("variant", [0, 8])
def test_zero_steps_is_a_noop(variant):
    """nsteps = 0 leaves the state (ghosts included) bitwise untouched; negative nsteps and a
    non-finite dt are rejected."""
    P, C = _mods()
    n = (40, 24, 32)
    h = tuple(2 * math.pi / v for v in n)
    g = P.Grid(C.SYS_WAVE, n, h)
    g.set_kernel_variant(variant)
    g.set_initial(C.INIT_NOISE, seed=5)
    before = g.get_state(padded=True)
    g.rk4_step(0.1, 0)
    assert np.array_equal(g.get_state(padded=True), before)
    with pytest.raises(C.ChemoraError):
        g.rk4_step(0.1, -1)
    with pytest.raises(C.ChemoraError):
        g.rk4_step(float("nan"), 1)


def test_stream_ordered_upload_download():
    """chemora_upload_state / chemora_download_state (pinned, no synchronisation) give the same
    state, ghosts and step result as chemora_set_initial(HOST) / chemora_get_state, also with
    two grids alternating on two streams."""
    P, C = _mods()
    import torch
    n = (40, 24, 32)
    h = tuple(2 * math.pi / v for v in n)
    y0 = ci.noise(n, 5, seed=8)
    ref = P.Grid(C.SYS_WAVE, n, h)
    ref.set_initial(C.INIT_HOST, y0)
    ref_pad0 = ref.get_state(padded=True)
    ref.rk4_step(0.1, 1)
    want = ref.get_state()
    grids = [P.Grid(C.SYS_WAVE, n, h) for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    hin = torch.from_numpy(y0).pin_memory()
    outs = [torch.empty(y0.shape, dtype=torch.float64).pin_memory() for _ in range(2)]
    for b in range(2):
        with torch.cuda.stream(streams[b]):
            grids[b].upload_state(hin)
            if b == 0:
                pad = grids[b].get_state(padded=True)
            grids[b].rk4_step(0.1, 1)
            grids[b].download_state(outs[b])
    torch.cuda.synchronize()
    assert np.array_equal(pad, ref_pad0)
    for b in range(2):
        assert np.array_equal(outs[b].numpy(), want)

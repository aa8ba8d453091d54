"""GPU tests of the temporally blocked wave step (kernel variant 8, wave_fused3.cu, 32x8
tiles): stages 1+2 and 3+4 each in one kernel with the intermediate state kept in shared
memory and registers.  They must give
bit-identical states to the one-kernel-per-stage path and match the oracle."""
from __future__ import annotations

import math

import numpy as np
import pytest

import chemora_inputs as ci
import oracle

pytestmark = pytest.mark.gpu
FUSED_VARIANTS = [8]


def _mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1410_1764_b200 as P
    from paper_1410_1764_b200 import capi as C
    return P, C


def _run(n, variant, steps, seed=2, ghost=3, order=4):
    P, C = _mods()
    h = tuple(2 * math.pi / v for v in n)
    g = P.Grid(C.SYS_WAVE, n, h, ghost=ghost, fd_order=order)
    g.set_kernel_variant(variant)
    g.set_initial(C.INIT_NOISE, seed=seed)
    g.rk4_step(0.25 * min(h), steps)
    return g, h


@pytest.mark.parametrize("fv", FUSED_VARIANTS)
@pytest.mark.parametrize("n", [(70, 45, 33), (64, 64, 64), (33, 17, 40), (8, 8, 8), (40, 37, 20)])
@pytest.mark.parametrize("steps", [1, 2, 3])
def test_fused_bitwise_equal_to_stagewise(n, steps, fv):
    a, _ = _run(n, 0, steps)
    b, _ = _run(n, fv, steps)
    assert np.array_equal(a.get_state(), b.get_state())
    assert np.array_equal(a.get_state(padded=True), b.get_state(padded=True))


@pytest.mark.parametrize("n", [(70, 45, 33), (33, 17, 40), (8, 8, 8), (40, 37, 20)])
@pytest.mark.parametrize("ghost", [1, 3])
def test_fused_order2_bitwise_equal_to_stagewise(n, ghost):
    """The same stage-pair kernels at stencil radius 1 (FD order 2; NEXT-1): odd radius, so
    the x-extended boxes carry an unused column for the TMA alignment; a ghost width of 1
    in the API keeps 2 in storage."""
    a, _ = _run(n, 0, 3, ghost=ghost, order=2)
    b, _ = _run(n, 8, 3, ghost=ghost, order=2)
    assert b.kernel_variant() == 8
    assert np.array_equal(a.get_state(), b.get_state())
    assert np.array_equal(a.get_state(padded=True), b.get_state(padded=True))


@pytest.mark.parametrize("n", [(70, 45, 33), (33, 17, 40), (12, 12, 12), (40, 37, 20)])
def test_fused_order6_bitwise_equal_to_stagewise(n):
    """The stage pairs at stencil radius 3 (FD order 6): storage ghost 6, the shallowest
    rings that fit shared memory, warps synchronised per iteration."""
    a, _ = _run(n, 0, 3, ghost=3, order=6)
    b, _ = _run(n, 8, 3, ghost=3, order=6)
    assert b.kernel_variant() == 8
    assert np.array_equal(a.get_state(), b.get_state())
    assert np.array_equal(a.get_state(padded=True), b.get_state(padded=True))


@pytest.mark.parametrize("fv", FUSED_VARIANTS)
def test_fused_parity_10_steps(fv):
    n = (48, 40, 56)
    P, C = _mods()
    h = tuple(2 * math.pi / v for v in n)
    dt = 0.25 * min(h)
    y0 = ci.pw3(n, h)
    g = P.Grid(C.SYS_WAVE, n, h)
    g.set_kernel_variant(fv)
    assert g.kernel_variant() == fv
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(dt, 10)
    ref = oracle.rk4(oracle.WAVE, y0, h, dt, 10)
    got = g.get_state()
    err = max(np.abs(got[f] - ref[f]).max() / np.abs(ref[f]).max() for f in range(5))
    assert err <= 1e-12
    nref = oracle.norms(oracle.WAVE, ref, h)
    np.testing.assert_allclose(g.norms(), nref, rtol=1e-12, atol=1e-12 * np.abs(nref).max())


@pytest.mark.parametrize("fv", FUSED_VARIANTS)
def test_fused_ghosts_and_variant_switch(fv):
    """Ghosts of the (rotated) state set are the periodic fill; switching back to the
    stage-wise kernels mid-run continues from the right set."""
    n = (40, 24, 32)
    a, h = _run(n, 0, 5)
    b, _ = _run(n, fv, 3)
    b.set_kernel_variant(0)
    b.rk4_step(0.25 * min(h), 2)
    assert np.array_equal(a.get_state(), b.get_state())
    pad = b.get_state(padded=True)
    ref = np.pad(pad[:, 3:-3, 3:-3, 3:-3], ((0, 0), (3, 3), (3, 3), (3, 3)), mode="wrap")
    assert np.array_equal(pad, ref)


@pytest.mark.parametrize("fv", FUSED_VARIANTS)
@pytest.mark.parametrize("nslabs", [2, 4])
def test_fused_local_slabs(nslabs, fv):
    P, C = _mods()
    n = (36, 20, 64)
    h = tuple(2 * math.pi / v for v in n)
    y0 = ci.noise(n, 5, seed=11)
    g = P.Grid(C.SYS_WAVE, n, h)
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(0.25 * min(h), 3)
    s = P.LocalSlabs(C.SYS_WAVE, n, h, nslabs)
    for gg in s.grids:
        gg.set_kernel_variant(fv)
    s.set_initial(C.INIT_HOST, y0)
    s.rk4_step(0.25 * min(h), 3)
    assert np.array_equal(s.get_state(), g.get_state())


@pytest.mark.parametrize("fv", FUSED_VARIANTS)
def test_fused_nonfinite_reported(fv):
    P, C = _mods()
    n = (16, 16, 16)
    h = (2 * math.pi / 16,) * 3
    y0 = ci.noise(n, 5, seed=1)
    y0[3, 4, 5, 6] = np.inf
    g = P.Grid(C.SYS_WAVE, n, h)
    g.set_kernel_variant(fv)
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(0.1, 2)
    with pytest.raises(C.ChemoraError) as ei:
        g.get_state()
    assert ei.value.code == C.E_NONFINITE

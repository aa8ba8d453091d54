"""GPU tests of the SURVEY.md §8(f) NEXT rows built this round: the fused energy monitor
(NEXT-3, Fig. 1 "Energy") and the model-driven tiling choice (NEXT-4,
PAPER.md:419-422, 578-582).  NEXT-1 (fd order) is in test_gpu_wave.py, NEXT-2 (fission)
in test_gpu_bssn.py / bench."""
from __future__ import annotations

import math

import numpy as np
import pytest

import chemora_inputs as ci
import oracle

pytestmark = pytest.mark.gpu


def _mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1410_1764_b200 as P
    from paper_1410_1764_b200 import capi as C
    return P, C


@pytest.mark.parametrize("variant", [0, 8])
@pytest.mark.parametrize("n", [(32, 32, 32), (70, 45, 33)])
def test_fused_energy_monitor_matches_oracle(n, variant):
    """Energy of the state after every step, reduced inside the kernel that writes the new
    state (stage-4 kernel, variant 0; stage-pair kernel B, variant 8), equals the oracle's
    energy of the oracle's state (1e-12) and the stand-alone norm (1e-13); the state itself
    is bitwise unchanged by monitoring."""
    P, C = _mods()
    h = tuple(2 * math.pi / v for v in n)
    dt = 0.25 * min(h)
    y0 = ci.noise(n, 5, seed=21)
    g = P.Grid(C.SYS_WAVE, n, h)
    g.set_kernel_variant(variant)
    g.set_initial(C.INIT_HOST, y0)
    g.set_monitor(True)
    assert g.kernel_variant() == variant
    g.rk4_step(dt, 4)
    e = g.read_monitor()
    assert len(e) == 4
    y = y0
    for s in range(4):
        y = oracle.rk4(oracle.WAVE, y, h, dt, 1)
        assert e[s] == pytest.approx(oracle.norms(oracle.WAVE, y, h)[-1], rel=1e-12)
    assert e[-1] == pytest.approx(g.norms()[-1], rel=1e-13)
    assert np.all(np.diff(e) <= 1e-15 * e[0])  # RK4 energy is non-increasing
    ref = P.Grid(C.SYS_WAVE, n, h)
    ref.set_initial(C.INIT_HOST, y0)
    ref.rk4_step(dt, 4)
    assert np.array_equal(ref.get_state(), g.get_state())
    # reading again returns nothing new; determinism across runs
    assert len(g.read_monitor()) == 0
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(dt, 4)
    assert np.array_equal(g.read_monitor(), e)


@pytest.mark.parametrize("order", [2, 6])
def test_fused_energy_monitor_other_orders(order):
    """The monitor instantiation of the stage-pair kernel B at stencil radius 1 and 3: the
    energy after every step equals the oracle's energy of the oracle's state at that order,
    and the state is bitwise the unmonitored one."""
    P, C = _mods()
    n = (40, 36, 44)
    h = tuple(2 * math.pi / v for v in n)
    dt = 0.2 * min(h)
    y0 = ci.noise(n, 5, seed=30 + order)
    g = P.Grid(C.SYS_WAVE, n, h, fd_order=order)
    assert g.kernel_variant() == 8
    g.set_initial(C.INIT_HOST, y0)
    g.set_monitor(True)
    g.rk4_step(dt, 3)
    e = g.read_monitor()
    y = y0
    for s in range(3):
        y = oracle.rk4(oracle.WAVE, y, h, dt, 1, g=order // 2, order=order)
        assert e[s] == pytest.approx(oracle.norms(oracle.WAVE, y, h, g=order // 2)[-1], rel=1e-12)
    ref = P.Grid(C.SYS_WAVE, n, h, fd_order=order)
    ref.set_initial(C.INIT_HOST, y0)
    ref.rk4_step(dt, 3)
    assert np.array_equal(ref.get_state(), g.get_state())


def test_dynamic_item_schedule_is_deterministic():
    """The temporally blocked wave kernels hand out their (tile, z-chunk) items dynamically
    (an atomic counter): which CTA runs which item changes from run to run.  On a grid with
    ~8 items per CTA the state stays bitwise equal to the one-kernel-per-stage path and the
    fused energy monitor (per-item partials, fixed-order sum) is bitwise reproducible."""
    P, C = _mods()
    n = (96, 96, 128)
    h = tuple(2 * math.pi / v for v in n)
    dt = 0.25 * min(h)
    y0 = ci.noise(n, 5, seed=33)
    ref = P.Grid(C.SYS_WAVE, n, h)
    ref.set_kernel_variant(0)
    ref.set_initial(C.INIT_HOST, y0)
    ref.rk4_step(dt, 3)
    g = P.Grid(C.SYS_WAVE, n, h)
    g.set_kernel_variant(8)
    g.set_monitor(True)
    runs = []
    for _ in range(3):
        g.set_initial(C.INIT_HOST, y0)
        g.rk4_step(dt, 3)
        runs.append(g.read_monitor())
        assert np.array_equal(g.get_state(), ref.get_state())
    assert all(np.array_equal(r, runs[0]) for r in runs[1:])
    assert runs[0][-1] == pytest.approx(ref.norms()[-1], rel=1e-13)


@pytest.mark.parametrize("system", ["wave", "bssn"])
def test_autotune_keeps_state_and_parity(system):
    """The autotuner times stage-1 launches with dt = 0 (state untouched) and keeps the
    fastest candidate; stepping afterwards still matches the oracle."""
    P, C = _mods()
    if system == "wave":
        n = (160, 96, 64)
        h = tuple(2 * math.pi / v for v in n)
        y0 = ci.noise(n, 5, seed=3)
        g = P.Grid(C.SYS_WAVE, n, h)
        sysid, params = oracle.WAVE, None
    else:
        n = (24, 24, 24)
        h = tuple(1.0 / v for v in n)
        y0 = ci.mink_pert(n, h, 1410)
        g = P.Grid(C.SYS_BSSN, n, h)
        sysid, params = oracle.BSSN, oracle.default_bssn_params()
    g.set_initial(C.INIT_HOST, y0)
    res = g.autotune(trials=2)
    assert res["candidates"] >= 2 and len(res["ms"]) == res["candidates"]
    assert np.array_equal(g.get_state(), y0)
    dt = 0.25 * min(h)
    g.rk4_step(dt, 2)
    ref = oracle.rk4(sysid, y0, h, dt, 2, params)
    err = max(np.abs(g.get_state()[f] - ref[f]).max() / max(np.abs(ref[f]).max(), 1e-6) for f in range(len(y0)))
    assert err <= 1e-10


@pytest.mark.parametrize("variant", [0, 8])
@pytest.mark.parametrize("nslabs", [2, 4])
def test_energy_monitor_local_slabs(nslabs, variant):
    """Per-slab fused monitors summed over the slabs (chemora_rk4_step_multi) give the
    oracle's energy; the state is still bitwise the single-grid state."""
    P, C = _mods()
    n = (36, 20, 64)
    h = tuple(2 * math.pi / v for v in n)
    dt = 0.25 * min(h)
    y0 = ci.noise(n, 5, seed=33)
    s = P.LocalSlabs(C.SYS_WAVE, n, h, nslabs)
    for g in s.grids:
        g.set_kernel_variant(variant)
    s.set_monitor(True)
    s.set_initial(C.INIT_HOST, y0)
    s.rk4_step(dt, 3)
    e = s.read_monitor()
    assert len(e) == 3
    y = y0
    for k in range(3):
        y = oracle.rk4(oracle.WAVE, y, h, dt, 1)
        assert e[k] == pytest.approx(oracle.norms(oracle.WAVE, y, h)[-1], rel=1e-12)
    ref = P.Grid(C.SYS_WAVE, n, h)
    ref.set_initial(C.INIT_HOST, y0)
    ref.rk4_step(dt, 3)
    assert np.array_equal(s.get_state(), ref.get_state())


@pytest.mark.parametrize("variant", [4, 3])
def test_bssn_constraint_monitor_matches_oracle(variant):
    """NEXT-3 for BSSN: with the monitor on, every step's stage-1 kernel
    reduces [L2, Linf] of H, M^i, G^i of the state entering the step (design 4: fused, from the
    on-chip derivatives; design 3: the constraint kernel before stage 1).  Equal to the oracle's
    constraints of the oracle's state after s = 0, 1, 2 steps (1e-10 of each norm, R11), and
    the monitored step is bitwise the unmonitored one."""
    P, C = _mods()
    n = (28, 20, 24)
    h = tuple(1.0 / v for v in n)
    dt = 0.25 * min(h)
    y0 = ci.mink_pert(n, h, 1410, eps=1e-2)
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_kernel_variant(variant)
    g.set_initial(C.INIT_HOST, y0)
    g.set_monitor(True)
    g.rk4_step(dt, 3)
    m = g.read_monitor()
    assert m.shape == (3, 14)
    vol = h[0] * h[1] * h[2]
    y = y0
    for s in range(3):
        c = oracle.constraints(y, h)
        ref = np.array([[math.sqrt(vol * (c[q] ** 2).sum()), np.abs(c[q]).max()] for q in range(7)]).ravel()
        np.testing.assert_allclose(m[s], ref, rtol=1e-10, atol=1e-10 * np.abs(ref).max())
        y = oracle.rk4(oracle.BSSN, y, h, dt, 1)
    r = P.Grid(C.SYS_BSSN, n, h)
    r.set_kernel_variant(variant)
    r.set_initial(C.INIT_HOST, y0)
    r.rk4_step(dt, 3)
    assert np.array_equal(r.get_state(), g.get_state())
    assert len(g.read_monitor()) == 0

"""GPU parity of the BSSN constraint monitors (R16):
chemora_constraints' fields and norms vs the oracle's constraint fields on the same state,
element by element (max |gpu - oracle| / max |oracle| per constraint, R11 norm)."""
from __future__ import annotations

import math

import numpy as np
import pytest

import chemora_inputs as ci
import oracle
from tests import bssn_exact

pytestmark = pytest.mark.gpu
B = 2
IX = {n: i for i, n in enumerate(ci.BSSN_GF)}


def _mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1410_1764_b200 as P
    from paper_1410_1764_b200 import capi as C
    return P, C


def _relerr(a, b):
    top = max(np.abs(b[q]).max() for q in range(b.shape[0]))
    out = []
    for q in range(a.shape[0]):
        s = max(np.abs(b[q]).max(), 1e-6 * top)
        out.append(np.abs(a[q] - b[q]).max() / s)
    return max(out)


def _norms_of(fields, h):
    vol = h[0] * h[1] * h[2]
    out = np.zeros(14)
    for q in range(7):
        out[2 * q] = math.sqrt(vol * float(np.sum(fields[q] ** 2)))
        out[2 * q + 1] = np.abs(fields[q]).max()
    return out


@pytest.mark.parametrize("n", [(20, 12, 12), (37, 21, 18)])
def test_constraint_fields_parity_mink_pert(n):
    P, C = _mods()
    h = tuple(1.0 / v for v in n)
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_initial(C.INIT_MINK_PERT, kind_params=[1e-2], seed=3)
    y = g.get_state()
    f = g.constraints().cpu().numpy()
    ref = oracle.constraints(y, h)
    assert np.abs(ref[0]).max() > 1e-3          # the data violate the constraints
    assert _relerr(f, ref) <= 1e-10
    nm = g.constraint_norms()
    assert np.allclose(nm, _norms_of(ref, h), rtol=1e-10, atol=0)


def test_constraint_fields_parity_pure_gauge_after_steps():
    """Strongly curved coordinates (pure-gauge exact solution), after 3 RK4 steps on the GPU:
    the GPU constraints of the GPU state equal the oracle's constraints of that state."""
    P, C = _mods()
    N = 24
    L = 2 * math.pi
    h = (L / N,) * 3
    n = (N, N, N)
    z, yy, x = ci.coords(n, h)
    x, yy, z = np.broadcast_arrays(x, yy, z)
    v = bssn_exact.bssn_vars(0.4, x, yy, z)
    st = np.zeros((25,) + x.shape)
    for nm, arr in v.items():
        st[IX[nm]] = arr
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_initial(C.INIT_HOST, st)
    g.rk4_step(0.25 * h[0], 3)
    y = g.get_state()
    f = g.constraints().cpu().numpy()
    ref = oracle.constraints(y, h)
    assert _relerr(f, ref) <= 1e-10


def test_constraints_flat_is_zero_and_wave_unsupported():
    P, C = _mods()
    n = (16, 12, 12)
    h = (0.1,) * 3
    g = P.Grid(C.SYS_BSSN, n, h)
    flat = np.zeros((25, n[2], n[1], n[0]))
    for nm in ("gt11", "gt22", "gt33", "alpha"):
        flat[IX[nm]] = 1.0
    g.set_initial(C.INIT_HOST, flat)
    assert np.abs(g.constraints().cpu().numpy()).max() == 0.0
    assert np.abs(g.constraint_norms()).max() == 0.0
    w = P.Grid(C.SYS_WAVE, n, h)
    with pytest.raises(C.ChemoraError):
        w.constraint_norms()


def test_constraint_norms_deterministic():
    P, C = _mods()
    n = (40, 24, 20)
    h = tuple(1.0 / v for v in n)
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_initial(C.INIT_MINK_PERT, kind_params=[1e-3], seed=9)
    g.rk4_step(0.25 * h[0], 2)
    a = g.constraint_norms()
    b = g.constraint_norms()
    assert np.array_equal(a, b)

"""Every BSSN kernel design (0: two-phase derivative-table kernel, 2: fissioned G1/G2/G3 kernels -- PAPER.md:537-547 fission; 3: HBM
derivative table + algebra kernels) matches
the oracle after RK4 steps, on ragged grids and at both gauges."""
from __future__ import annotations

import numpy as np
import pytest

import chemora_inputs as ci
import oracle

pytestmark = pytest.mark.gpu
BENCH = [2.0, 1.0, 1.0, 0.0, 1.0, 0.75, 0.0, 1.0, 1.0, 1.0]
HARMONIC = [1.0, 2.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0, 1.0]
GENERIC = [1.5, 2.0, 0.7, 0.3, 0.8, 0.6, 1.0, 0.5, 0.9, 0.7]


def _mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1410_1764_b200 as P
    from paper_1410_1764_b200 import capi as C
    return P, C


def relerr(a, b):
    top = max(np.abs(b[f]).max() for f in range(b.shape[0]))
    return max(np.abs(a[f] - b[f]).max() / max(np.abs(b[f]).max(), 1e-6 * top) for f in range(b.shape[0]))


@pytest.mark.parametrize("variant", [0, 2, 3, 4])
@pytest.mark.parametrize("params", [BENCH, HARMONIC, GENERIC])
def test_variant_parity(variant, params):
    P, C = _mods()
    n = (45, 22, 30)   # x not a multiple of the 32-point table tile
    h = tuple(1.0 / v for v in n)
    y0 = ci.mink_pert(n, h, 1410, eps=1e-2)
    y0[ci.BSSN_GF.index("alpha")] += 0.05
    g = P.Grid(C.SYS_BSSN, n, h, params=params)
    g.set_kernel_variant(variant)
    g.set_initial(C.INIT_HOST, y0)
    k = g.rhs().cpu().numpy()
    assert relerr(k, oracle.rhs(oracle.BSSN, y0, h, params)) <= 1e-10
    dt = 0.25 * min(h)
    g.rk4_step(dt, 3)
    ref = oracle.rk4(oracle.BSSN, y0, h, dt, 3, params)
    got = g.get_state()
    assert relerr(got, ref) <= 1e-10
    assert relerr(got - y0, ref - y0) <= 1e-8


@pytest.mark.parametrize("variant", [3, 4])
def test_nonfinite_reported_with_gf(variant):
    """A NaN injected into one GF (gt22) surfaces as CHEMORA_E_NONFINITE at the next
    synchronising call, naming the first offending GF and the step."""
    P, C = _mods()
    n = (16, 16, 16)
    h = tuple(1.0 / v for v in n)
    y0 = ci.mink_pert(n, h, 1410, eps=1e-3)
    y0[ci.BSSN_GF.index("gt22"), 3, 4, 5] = np.nan
    g = P.Grid(C.SYS_BSSN, n, h)
    g.set_kernel_variant(variant)
    g.set_initial(C.INIT_HOST, y0)
    g.rk4_step(0.25 * min(h), 1)
    with pytest.raises(C.ChemoraError) as ei:
        g.get_state()
    assert ei.value.code == C.E_NONFINITE
    msg = str(ei.value)
    assert "at step 0" in msg
    # the NaN spreads to every GF through the stencils; the flag keeps the lowest index
    assert "grid function 0" in msg

"""The BSSN derivative kernel (variant 3) marches z in per-CTA chunks (CHEMORA_BSSN_DZC,
default 32) with a cp.async plane ring primed per chunk, and the algebra kernels' register
caps are selectable per group (CHEMORA_BSSN_ALG_MB).  Neither may change a single bit of
the result: every chunk length -- shorter than the stencil radius, ragged against the slab,
longer than the slab -- and every cap must reproduce the default state exactly.  The knobs
are read once per process, so each setting runs in its own subprocess."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import chemora_inputs as ci
import paper_1410_1764_b200 as P
from paper_1410_1764_b200 import capi as C
n = (45, 22, 70)
h = tuple(1.0 / v for v in n)
y0 = ci.mink_pert(n, h, 1410, eps=1e-2)
g = P.Grid(C.SYS_BSSN, n, h)
g.set_kernel_variant(3)
g.set_initial(C.INIT_HOST, y0)
g.rk4_step(0.25 * min(h), 2)
np.save(sys.argv[1], g.get_state())
"""


def _run(tmp_dir, name, env_extra):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    out = tmp_dir / f"{name}.npy"
    env = dict(os.environ)
    env.pop("CHEMORA_BSSN_DZC", None)
    env.pop("CHEMORA_BSSN_ALG_MB", None)
    env.update(env_extra)
    subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), str(out)], check=True, env=env,
                   cwd=ROOT, timeout=600)
    return np.load(out)


@pytest.fixture(scope="module")
def default_state(tmp_path_factory):
    return _run(tmp_path_factory.mktemp("bssn_default"), "default", {})


@pytest.mark.parametrize("env", [{"CHEMORA_BSSN_DZC": "1"}, {"CHEMORA_BSSN_DZC": "2"},
                                 {"CHEMORA_BSSN_DZC": "7"}, {"CHEMORA_BSSN_DZC": "48"},
                                 {"CHEMORA_BSSN_DZC": "100"},
                                 {"CHEMORA_BSSN_ALG_MB": "33"}, {"CHEMORA_BSSN_ALG_MB": "23"}])
def test_bssn_chunking_and_caps_are_bitwise_neutral(tmp_path, default_state, env):
    ref = default_state
    got = _run(tmp_path, "probe", env)
    assert np.isfinite(ref).all()
    assert np.array_equal(got, ref), f"{env}: max diff {np.abs(got - ref).max()}"

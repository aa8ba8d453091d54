"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/chemora.h
declares, and validates descriptors (no compute calls: there is no GPU here)."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "chemora.h")
LIB = os.path.join(ROOT, "paper_1410_1764_b200", "libchemora.so")


def _ensure_built():
    if not os.path.exists(LIB):
        from paper_1410_1764_b200 import build as b
        b.build()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(chemora_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("chemora_grid_create", "chemora_set_initial", "chemora_rhs", "chemora_rk4_step",
              "chemora_halo_exchange", "chemora_norms"):
        assert n in names


def test_library_exports_every_declared_symbol():
    _ensure_built()
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    _ensure_built()
    from paper_1410_1764_b200 import capi
    assert set(declared_functions()) <= set(capi.EXPORTED)


def _desc(**kw):
    from paper_1410_1764_b200 import capi as C
    args = dict(system=C.SYS_WAVE, extent=(32, 32, 32), spacing=(0.1, 0.1, 0.1))
    args.update(kw)
    return C.make_desc(**args)


def test_required_bytes_layout():
    """4 sets x 5 GFs of padded arrays: Px = round_up(16 + N + gs, 16), Py = Pz = N + 2gs with
    the storage ghost gs = max(g, 4) of 4th-order wave grids."""
    _ensure_built()
    from paper_1410_1764_b200 import capi as C
    n = C.chemora_grid_required_bytes(_desc())
    px, py, pz = 64, 40, 40
    arr = ((px * py * pz + 31) // 32) * 32 * 8
    assert n >= 4 * 5 * arr
    assert n < 4 * 5 * arr + 300_000
    n512 = C.chemora_grid_required_bytes(_desc(extent=(512, 512, 512)))
    assert 23.0e9 < n512 < 23.8e9  # fits one B200 with room to spare
    # 2nd-order grids keep g = 3 (radius 1)
    n2 = C.chemora_grid_required_bytes(_desc(fd_order=2))
    assert n2 < n


@pytest.mark.parametrize("kw,code", [
    (dict(ghost=1), 2),                      # g below the 4th-order radius
    (dict(extent=(4, 32, 32)), 2),           # N < 2g
    (dict(nranks=3), 2),                     # Nz not divisible
    (dict(nranks=8, extent=(32, 32, 32)), 2),  # local slab 4 < 2g
    (dict(fd_order=5), 7),
    (dict(spacing=(0.1, -1.0, 0.1)), 1),
])
def test_descriptor_validation(kw, code):
    _ensure_built()
    from paper_1410_1764_b200 import capi as C
    with pytest.raises(C.ChemoraError) as ei:
        C.chemora_grid_required_bytes(_desc(**kw))
    assert ei.value.code == code
    assert C.chemora_last_error()


def test_bssn_needs_ghost3_and_n_gf():
    _ensure_built()
    from paper_1410_1764_b200 import capi as C
    with pytest.raises(C.ChemoraError):
        C.chemora_grid_required_bytes(_desc(system=C.SYS_BSSN, ghost=2))
    d = _desc(system=C.SYS_BSSN)
    d.n_gf = 5
    with pytest.raises(C.ChemoraError):
        C.chemora_grid_required_bytes(d)
    assert C.chemora_grid_required_bytes(_desc(system=C.SYS_BSSN)) > 0


def test_norms_combine_host_logic():
    """Rank-ordered combination: L2 = sqrt(h^3 sum), Linf = max, sum = h^3 sum."""
    _ensure_built()
    import numpy as np
    from paper_1410_1764_b200 import capi as C
    d = _desc(spacing=(0.5, 0.5, 0.5))
    L = C.chemora_norms_len(C.SYS_WAVE)
    assert L == 16
    parts = np.zeros((2, L))
    parts[0, 0], parts[1, 0] = 3.0, 5.0      # sum f^2
    parts[0, 1], parts[1, 1] = 2.0, 7.0      # max
    parts[0, 2], parts[1, 2] = -1.0, 4.0     # sum
    parts[:, 15] = [1.0, 2.0]                # energy
    out = C.chemora_norms_combine(d, parts, 2)
    assert out[0] == pytest.approx((0.125 * 8.0) ** 0.5)
    assert out[1] == 7.0
    assert out[2] == pytest.approx(0.125 * 3.0)
    assert out[15] == pytest.approx(0.125 * 3.0)


def test_combine_constraint_partials():
    """Rank-major constraint partials -> L2 = sqrt(h^3 sum), Linf = max over ranks."""
    _ensure_built()
    import numpy as np
    from paper_1410_1764_b200 import capi as C
    parts = np.zeros((2, 14))
    parts[0, 0::2] = np.arange(7) + 1.0
    parts[1, 0::2] = 2.0 * (np.arange(7) + 1.0)
    parts[0, 1::2] = 0.5
    parts[1, 1::2] = np.linspace(0.1, 0.9, 7)
    out = C.chemora_constraint_norms_combine(_desc(system=C.SYS_BSSN, spacing=(0.5, 0.5, 0.5)), parts, 2)
    assert np.allclose(out[0::2], np.sqrt(0.125 * 3.0 * (np.arange(7) + 1.0)), rtol=1e-15)
    assert np.array_equal(out[1::2], np.maximum(0.5, np.linspace(0.1, 0.9, 7)))


def test_missing_library_fails_loudly(tmp_path):
    """Without libchemora.so the binding refuses to import (there is no CPU fallback)."""
    import shutil
    import subprocess
    import sys
    src = os.path.join(ROOT, "paper_1410_1764_b200")
    shutil.copytree(src, tmp_path / "paper_1410_1764_b200",
                    ignore=shutil.ignore_patterns("*.so", "build_obj", "csrc", "__pycache__"))
    r = subprocess.run([sys.executable, "-c", "import paper_1410_1764_b200.capi"], cwd=tmp_path,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "is missing" in r.stderr and "no CPU fallback" in r.stderr


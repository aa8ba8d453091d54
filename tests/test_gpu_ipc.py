"""Cross-process peer records (chemora_grid_export_peer): the record carries the
workspace's offset inside the CUDA allocation its IPC handle maps, so a workspace that a
caching allocator placed inside a larger block is opened at the right address.  (Opening the
handle needs a second process on another GPU; this checks the exported offset against the
driver's own cuMemGetAddressRange.)"""
from __future__ import annotations

import struct

import pytest

pytestmark = pytest.mark.gpu


def _mods():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1410_1764_b200 as P
    from paper_1410_1764_b200 import capi as C
    return P, C


@pytest.mark.parametrize("pad", [0, 1 << 20, 3 << 20])
def test_export_peer_records_workspace_offset(pad):
    P, C = _mods()
    import torch
    try:
        from cuda.bindings import driver as cu
    except ImportError:
        pytest.skip("cuda-python driver bindings unavailable")
    n = (16, 16, 32)
    desc = C.make_desc(C.SYS_WAVE, n, (0.1, 0.1, 0.1), nranks=2, rank=0)
    nbytes = C.chemora_grid_required_bytes(desc)
    big = torch.empty(nbytes + pad, dtype=torch.uint8, device="cuda")
    ws = big[pad:]
    h = C.chemora_grid_create(desc, ws.data_ptr(), nbytes)
    try:
        rec = C.chemora_grid_export_peer(h)
        (offset,) = struct.unpack_from("<Q", rec, 64)   # after the 64-byte cudaIpcMemHandle_t
        err, base, size = cu.cuMemGetAddressRange(ws.data_ptr())
        assert err == cu.CUresult.CUDA_SUCCESS
        assert offset == ws.data_ptr() - int(base)
        assert offset >= pad
    finally:
        C.chemora_grid_destroy(h)

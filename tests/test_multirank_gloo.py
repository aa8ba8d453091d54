"""World-size 2 and 3 CPU tests (gloo) of the multi-rank host logic: ring topology, slab
bounds, the peer-record exchange that connects neighbouring z-slabs, the host phase barrier,
and the C library's rank-ordered combination of per-rank partials.  (The device side of the
N>1 path -- stage kernels storing into peer ghost planes, the collective norms over peer
memory -- runs in tests/test_gpu_ipc_procs.py: 2 and 3 processes on one GPU.)"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = globals()[fn_name](rank, world)
        q.put((rank, out))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(world, fn_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _records(rank, world):
    from paper_1410_1764_b200 import dist as D
    rec = f"rank{rank}".encode() + b"\x00\x01" * 8  # opaque bytes with NULs
    lo, hi = D.exchange_records(rec, rank, world)
    return lo, hi


@pytest.mark.parametrize("world", [2, 3])
def test_peer_record_exchange_ring(world):
    res = _run(world, "_records")
    for r in range(world):
        lo, hi = res[r]
        assert lo.startswith(f"rank{(r - 1) % world}".encode())
        assert hi.startswith(f"rank{(r + 1) % world}".encode())
        assert lo.endswith(b"\x00\x01" * 8)
    if world == 2:  # both faces go to the same peer
        assert res[0][0] == res[0][1]


def _gather(part, world):
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, np.asarray(part, dtype=np.float64).tolist())
    return np.array(out, dtype=np.float64)


def _norms(rank, world):
    """Each rank owns a z-slab of one global field; partials computed here in numpy, then
    gathered and combined by the C library in rank order."""
    from paper_1410_1764_b200 import capi as C
    from paper_1410_1764_b200 import dist as D
    rng = np.random.default_rng(42)
    field = rng.standard_normal((5, 12, 6, 7))  # [gf][z][y][x], global
    z0, nz = D.slab_bounds(12, world, rank)
    sl = field[:, z0:z0 + nz]
    part = np.zeros(C.chemora_norms_len(C.SYS_WAVE))
    for f in range(5):
        part[3 * f] = (sl[f] ** 2).sum()
        part[3 * f + 1] = np.abs(sl[f]).max()
        part[3 * f + 2] = sl[f].sum()
    part[15] = 0.5 * (sl[1:] ** 2).sum()
    gathered = _gather(part, world)
    desc = C.make_desc(C.SYS_WAVE, (7, 6, 12), (0.5, 0.5, 0.5), rank=rank, nranks=world)
    combined = C.chemora_norms_combine(desc, gathered, world)
    return combined.tolist(), gathered[:, 0].tolist()


@pytest.mark.parametrize("world", [2, 3])
def test_norm_partials_combine_in_rank_order(world):
    res = _run(world, "_norms")
    rng = np.random.default_rng(42)
    field = rng.standard_normal((5, 12, 6, 7))
    vol = 0.125
    for r in range(world):
        combined, col = res[r]
        assert combined == res[0][0]  # every rank gets the identical result
        for f in range(5):
            assert combined[3 * f] == pytest.approx(np.sqrt(vol * (field[f] ** 2).sum()), rel=1e-14)
            assert combined[3 * f + 1] == np.abs(field[f]).max()
            assert combined[3 * f + 2] == pytest.approx(vol * field[f].sum(), rel=1e-12, abs=1e-14)
        assert combined[15] == pytest.approx(vol * 0.5 * (field[1:] ** 2).sum(), rel=1e-14)
        # rows are in rank order: rank r's row holds slab r's sum of squares
        for rr in range(world):
            z0, nz = (rr * 12 // world, 12 // world)
            assert col[rr] == pytest.approx((field[0, z0:z0 + nz] ** 2).sum(), rel=1e-14)


def _constraints(rank, world):
    """Constraint-monitor partials [sum c^2, max |c|] x 7 of each rank's slab, gathered and
    combined on every rank by chemora_constraint_norms_combine (the combine step of the
    collective chemora_constraint_norms)."""
    from paper_1410_1764_b200 import capi as C
    from paper_1410_1764_b200 import dist as D
    rng = np.random.default_rng(7)
    c = rng.standard_normal((7, 12, 5, 6))
    z0, nz = D.slab_bounds(12, world, rank)
    sl = c[:, z0:z0 + nz]
    part = np.zeros(14)
    for q in range(7):
        part[2 * q] = (sl[q] ** 2).sum()
        part[2 * q + 1] = np.abs(sl[q]).max()
    gathered = _gather(part, world)
    desc = C.make_desc(C.SYS_BSSN, (6, 5, 12), (0.25, 1.0, 1.0), rank=rank, nranks=world)
    return C.chemora_constraint_norms_combine(desc, gathered, world).tolist()


@pytest.mark.parametrize("world", [2, 3])
def test_constraint_partials_combine(world):
    res = _run(world, "_constraints")
    c = np.random.default_rng(7).standard_normal((7, 12, 5, 6))
    for r in range(world):
        assert res[r] == res[0]
        for q in range(7):
            assert res[r][2 * q] == pytest.approx(np.sqrt(0.25 * (c[q] ** 2).sum()), rel=1e-14)
            assert res[r][2 * q + 1] == np.abs(c[q]).max()


def test_slab_bounds_and_validation():
    from paper_1410_1764_b200 import capi as C
    from paper_1410_1764_b200 import dist as D
    for world in (1, 2, 4, 8):
        covered = []
        for r in range(world):
            z0, nz = D.slab_bounds(1024, world, r)
            covered.extend(range(z0, z0 + nz))
        assert covered == list(range(1024))
        d = C.make_desc(C.SYS_WAVE, (64, 64, 1024), (0.1,) * 3, rank=world - 1, nranks=world)
        assert C.chemora_grid_required_bytes(d) > 0
    with pytest.raises(ValueError):
        D.slab_bounds(1000, 3, 0)
    assert D.ring_neighbours(0, 4) == (3, 1)
    assert D.ring_neighbours(3, 4) == (2, 0)


def _barrier_cb(rank, world):
    """The phase-barrier callback the library calls between phases is a real barrier: no
    rank leaves round k before every rank has entered it."""
    import time
    import torch.distributed as dist
    from paper_1410_1764_b200 import dist as D
    cb = D.barrier_callback()
    seen = []
    for k in range(3):
        time.sleep(0.05 * ((rank + k) % world))
        t = time.time()
        cb(None)
        seen.append(t)
    allt = [None] * world
    dist.all_gather_object(allt, seen)
    return allt


@pytest.mark.parametrize("world", [2, 3])
def test_phase_barrier_callback(world):
    res = _run(world, "_barrier_cb")
    allt = res[0]
    # entry times of round k of every rank precede ... (ordering checked through exits:
    # each rank records its entry time; all ranks' round-k entries precede any round-(k+1) entry)
    for k in range(2):
        assert max(t[k] for t in allt) <= min(t[k + 1] for t in allt)

"""Multi-rank plumbing over torch.distributed (process groups only; no arithmetic of the
method): the z-slab ring topology (PAPER.md:200-204 driver decomposition), the exchange of
the per-rank peer records that connect neighbouring slabs, and the gather of per-rank norm
partials that the C library combines in rank order (chemora_norms_combine)."""
from __future__ import annotations

import numpy as np


def ring_neighbours(rank: int, world: int) -> tuple[int, int]:
    """(lower, upper) z-slab neighbours on the periodic ring."""
    return (rank - 1) % world, (rank + 1) % world


def slab_bounds(nz_global: int, world: int, rank: int) -> tuple[int, int]:
    """Global z index of local plane 0 and the local plane count (Nz must divide evenly,
    the C library validates the same rule)."""
    if nz_global % world:
        raise ValueError("extent[2] must be divisible by the number of ranks")
    nzl = nz_global // world
    return rank * nzl, nzl


def exchange_records(record: bytes, rank: int, world: int, group=None) -> tuple[bytes, bytes]:
    """all_gather the opaque peer records; return the (lower, upper) neighbours' records."""
    import torch.distributed as dist
    allrec = [None] * world
    dist.all_gather_object(allrec, record, group=group)
    lo, hi = ring_neighbours(rank, world)
    return allrec[lo], allrec[hi]


def gather_partials(partials: np.ndarray, world: int, group=None) -> np.ndarray:
    """all_gather per-rank norm partials; rows in rank order (deterministic combine)."""
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, np.asarray(partials, dtype=np.float64).tolist(), group=group)
    return np.array(out, dtype=np.float64)


def combine_constraint_partials(gathered: np.ndarray, vol: float) -> np.ndarray:
    """Rank-major [world][14] partials [sum c_q^2, max |c_q|] x 7 of chemora_constraints ->
    [L2_q, Linf_q] x 7 (sums in rank order, so the result is deterministic)."""
    g = np.asarray(gathered, dtype=np.float64).reshape(-1, 14)
    out = np.zeros(14)
    for q in range(7):
        s = 0.0
        for r in range(g.shape[0]):
            s += g[r, 2 * q]
        out[2 * q] = np.sqrt(vol * s)
        out[2 * q + 1] = g[:, 2 * q + 1].max()
    return out


def sum_in_rank_order(gathered: np.ndarray) -> np.ndarray:
    """Rank-major [world][n] per-slab values (e.g. monitor energies) -> their sums over the
    slabs, added in rank order (deterministic)."""
    g = np.asarray(gathered, dtype=np.float64)
    if g.ndim == 1:
        g = g[:, None]
    out = np.zeros(g.shape[1])
    for r in range(g.shape[0]):
        out = out + g[r]
    return out

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

"""Multi-rank plumbing over torch.distributed (process groups only; no arithmetic of the
method): the z-slab ring topology (PAPER.md:200-204 driver decomposition), the exchange of
the opaque per-rank peer records that connect neighbouring slabs, and the host barrier the
library calls between phases when ranks share one device.  Every reduction over ranks
(norms, constraint norms, monitor energies) is done by the C library itself
(chemora_norms & co. are collective over the peer-mapped workspaces)."""
from __future__ import annotations


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


def barrier_callback(group=None):
    """The host barrier chemora_set_phase_barrier calls after every phase."""
    import torch.distributed as dist

    def _barrier(_user):
        dist.barrier(group=group)
    return _barrier

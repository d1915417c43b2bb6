"""Slab decomposition of the outermost grid axis, host side.

The device keeps, per rank, its owned node planes [k_begin, k_end) plus one ghost
plane on each interior face; after every pseudo-time step rank r sends its first
owned plane to r-1 and its last to r+1 and receives their boundary planes into its
ghosts (csrc/petto_dev.cu: halo()).  This module holds the same bookkeeping for the
Python callers (bench.py under torchrun) and for the CPU tests that check the
schedule with torch.distributed/gloo.
"""
from __future__ import annotations


def slab_range(rank: int, nranks: int, nz: int):
    """Balanced contiguous split of nz planes: [k_begin, k_end) of `rank`."""
    if not 0 <= rank < nranks or nranks > nz:
        raise ValueError("slab: need 0 <= rank < nranks <= nz")
    base, extra = divmod(nz, nranks)
    kb = rank * base + min(rank, extra)
    return kb, kb + base + (1 if rank < extra else 0)


def stored_range(rank: int, nranks: int, nz: int):
    """Planes a rank keeps in HBM: owned plus one ghost per interior face."""
    kb, ke = slab_range(rank, nranks, nz)
    return max(0, kb - 1), min(nz, ke + 1)


def halo_schedule(rank: int, nranks: int, nz: int):
    """(peer, plane sent, plane received) for one exchange, lower neighbour first."""
    kb, ke = slab_range(rank, nranks, nz)
    out = []
    if rank > 0:
        out.append((rank - 1, kb, kb - 1))
    if rank < nranks - 1:
        out.append((rank + 1, ke - 1, ke))
    return out


def exchange_numpy(planes: dict, rank: int, nranks: int, nz: int, dist) -> None:
    """Apply halo_schedule to {plane index: ndarray} with torch.distributed p2p
    (gloo on CPU).  Sends are posted before receives to avoid ordering deadlocks."""
    import numpy as np
    import torch

    reqs = []
    for peer, send_k, _ in halo_schedule(rank, nranks, nz):
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(planes[send_k])), peer))
    for peer, _, recv_k in halo_schedule(rank, nranks, nz):
        buf = torch.empty(planes[recv_k].shape, dtype=torch.float64)
        dist.recv(buf, peer)
        planes[recv_k][...] = buf.numpy()
    for r in reqs:
        r.wait()

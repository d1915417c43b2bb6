"""CPU: the slab decomposition bookkeeping (paper_2509_06971_b200/slab.py, the same
schedule as csrc/petto_dev.cu halo()) with torch.distributed/gloo, world size 2 and
3: a 27-point stencil stepped on ghosted slabs equals the global computation."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_06971_b200 import slab


def test_slab_ranges_partition_the_axis():
    for nz in (3, 7, 64, 256):
        for n in range(1, min(nz, 9) + 1):
            ranges = [slab.slab_range(r, n, nz) for r in range(n)]
            assert ranges[0][0] == 0 and ranges[-1][1] == nz
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert max(e - b for b, e in ranges) - min(e - b for b, e in ranges) <= 1
            for r in range(n):
                s0, s1 = slab.stored_range(r, n, nz)
                kb, ke = ranges[r]
                assert s0 == max(0, kb - 1) and s1 == min(nz, ke + 1)


def stencil27(u, k0, k1):
    """Mean over the 3x3x3 neighbourhood (clamped at the grid ends) for planes k0..k1-1."""
    nz, ny, nx = u.shape
    out = np.zeros((k1 - k0, ny, nx))
    p = np.pad(u, ((0, 0), (1, 1), (1, 1)), mode="edge")
    for dk in (-1, 0, 1):
        kk = np.clip(np.arange(k0, k1) + dk, 0, nz - 1)
        for dj in range(3):
            for di in range(3):
                out += p[kk, dj:dj + ny, di:di + nx]
    return out / 27.0


def worker(rank, n, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    nz, ny, nx, steps = 11, 6, 5, 4
    g = np.random.default_rng(0).random((nz, ny, nx))
    kb, ke = slab.slab_range(rank, n, nz)
    s0, s1 = slab.stored_range(rank, n, nz)
    local = {k: g[k].copy() for k in range(s0, s1)}
    for _ in range(steps):
        arr = np.stack([local[k] for k in range(s0, s1)])
        # a stencil over the stored planes, kept for the owned planes only
        full = np.zeros((nz, ny, nx))
        full[s0:s1] = arr
        new = stencil27(full, kb, ke) if s0 == 0 and s1 == nz else None
        if new is None:
            # emulate clamping at physical ends only: ghosts stand in for interior neighbours
            new = np.zeros((ke - kb, ny, nx))
            p = np.pad(full, ((0, 0), (1, 1), (1, 1)), mode="edge")
            for dk in (-1, 0, 1):
                kk = np.clip(np.arange(kb, ke) + dk, 0, nz - 1)
                for dj in range(3):
                    for di in range(3):
                        new += p[kk, dj:dj + ny, di:di + nx]
            new /= 27.0
        for k in range(kb, ke):
            local[k] = new[k - kb]
        slab.exchange_numpy(local, rank, n, nz, dist)
    want = g.copy()
    for _ in range(steps):
        want = stencil27(want, 0, nz)
    err = max(float(np.abs(local[k] - want[k]).max()) for k in range(s0, s1))
    q.put((rank, err))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [2, 3])
def test_halo_schedule_gloo(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + n
    procs = [ctx.Process(target=worker, args=(r, n, port, q)) for r in range(n)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(n)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err in res:
        assert err == 0.0, (rank, err)

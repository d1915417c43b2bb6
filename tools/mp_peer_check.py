"""Multi-process check of the peer halo (CUDA IPC + cross-process stream flags).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29611 tools/mp_peer_check.py [--device 0]

Every rank owns a z slab of a C4-shaped cantilever problem, exports / imports the
peer blobs over gloo, runs two hybrid solves (with a state upload in between)
and sends its owned planes to rank 0, which compares them bit for bit with a
single-context solve.  With one GPU all ranks share it (no kernel waits on
another rank; only streams wait on flags).
"""
import argparse
import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_06971_b200 import device as D  # noqa: E402
from paper_2509_06971_b200 import problem as P  # noqa: E402
from paper_2509_06971_b200 import slab  # noqa: E402


def main():
    a = argparse.ArgumentParser()
    a.add_argument("--device", type=int, default=None)
    args = a.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = args.device if args.device is not None else int(os.environ.get("LOCAL_RANK", 0))
    dist.init_process_group("gloo")
    cfg = P.config("C4")
    prob = P.build_problem(cfg)
    g = prob.grid
    rng = np.random.default_rng(5)
    E = rng.uniform(0.2, 1.0, g.num_nodes)
    s0 = rng.uniform(-1e-3, 1e-3, 3 * g.num_nodes)
    s1 = rng.uniform(-1e-3, 1e-3, 3 * g.num_nodes)
    sched = P.build_schedule(cfg, g, spectral_bound=D.spectral_bound)
    p = P.PTParams(sched.pt.dt_pt, sched.pt.dt_apt, 1.0, 40, 7, 1)

    def setup(ctx):
        ctx.set_constraints(prob.cons_entry, prob.cons_value)
        ctx.set_source(prob.source)
        ctx.set_property(E)
        ctx.init_operator()
        ctx.set_state(s0, s0)

    kr = slab.slab_range(rank, world, g.n[2])
    ctx = D.Context(g, 1, prob.poisson_ratio, D.MODE_FAST, device=dev, k_range=kr)
    setup(ctx)
    blobs = [None] * world
    dist.all_gather_object(blobs, ctx.peer_export())
    ctx.peer_import(blobs[rank - 1] if rank > 0 else None, blobs[rank + 1] if rank + 1 < world else None)
    dist.barrier()
    ctx.hybrid_solve(p)
    ctx.set_state(s1, s0)
    ctx.hybrid_solve(p)
    cur = np.full(3 * g.num_nodes, np.nan)
    prev = np.full(3 * g.num_nodes, np.nan)
    ctx.get_state(cur, prev)
    parts = [None] * world
    dist.all_gather_object(parts, (kr, cur, prev))
    ok = True
    if rank == 0:
        one = D.Context(g, 1, prob.poisson_ratio, D.MODE_FAST, device=dev)
        setup(one)
        one.hybrid_solve(p)
        one.set_state(s1, s0)
        one.hybrid_solve(p)
        want_c, want_p = one.get_state()
        plane = g.n[0] * g.n[1]
        for (k0, k1), c, pv in parts:
            for comp in range(3):
                sl = slice(comp * g.num_nodes + k0 * plane, comp * g.num_nodes + k1 * plane)
                ok &= np.array_equal(c[sl], want_c[sl]) and np.array_equal(pv[sl], want_p[sl])
        print(f"peer halo, {world} processes: {'bit-identical' if ok else 'MISMATCH'}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())

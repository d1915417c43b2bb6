"""TEST INFRASTRUCTURE: the slab decomposition in its deployment shape -- one
PROCESS per rank under torchrun -- with several ranks on one GPU, through the
multi-process NCCL emulator (tests/nccl_emu/nccl_emu_mp.cu):

    PETTO_NCCL_LIB=tests/nccl_emu/libnccl_emu_mp.so python -m torch.distributed.run \\
        --nnodes 1 --nproc-per-node N --master-addr 127.0.0.1 --master-port P \\
        tests/nccl_emu/run_ranks_mp.py replica|fast z|x nccl|peer

torch.distributed (gloo) carries only the set-up (unique id, peer-halo IPC blobs)
and the gathering of the results; every exchange of the solver goes through the
library's NCCL branches (ghost planes by send/recv, or by the fused kernel's peer
stores over CUDA IPC), all-reduced scalars, the REPLICA chain, broadcasts.  The
sequence per rank is run_ranks.py's: hybrid_solve, residual norm,
iterate_to_tolerance, a 3-loop run().  Rank 0 prints one JSON line comparing the
gathered results with the single-domain context."""
import json
import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2509_06971_b200 import device as D  # noqa: E402
from paper_2509_06971_b200 import problem as P  # noqa: E402
from paper_2509_06971_b200 import slab  # noqa: E402

mode = D.MODE_REPLICA if sys.argv[1] == "replica" else D.MODE_FAST
xo = sys.argv[2] == "x"
halo = sys.argv[3]
dist.init_process_group("gloo")
rank, nranks = dist.get_rank(), dist.get_world_size()
cfg = P.config("C4", nx=40, ny=14, nz=13, n_apt=30, n_pt=30, max_loops=3, report_every=1)
prob = P.build_problem(cfg)
g = prob.grid
N = g.num_nodes
sched = P.build_schedule(cfg, g, spectral_bound=D.spectral_bound)
axis = 0 if xo else 2
rng = np.random.default_rng(5)
u0 = rng.uniform(-1e-3, 1e-3, 3 * N)
E = np.maximum(1e-6, rng.random(N) ** 3)
p_solve = P.PTParams(sched.pt.dt_pt, sched.pt.dt_apt, sched.pt.theta, 37, 11, sched.pt.form)


def setup_solver(ctx):
    ctx.set_constraints(prob.cons_entry, prob.cons_value)
    ctx.set_source(prob.source)
    ctx.set_property(E)
    ctx.init_operator()
    ctx.set_state(u0, u0)


def join(ctx):
    """NCCL communicator (and the peer halo) of one set of slab contexts."""
    uid = [D.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, 0)
    ctx.comm_init(uid[0], rank, nranks)
    if halo == "peer":
        blobs = [None] * nranks
        dist.all_gather_object(blobs, ctx.peer_export())
        ctx.peer_import(blobs[rank - 1] if rank > 0 else None, blobs[rank + 1] if rank + 1 < nranks else None)


def work(ctx, run_ctx, phases_buf=None):
    out = {}
    ctx.hybrid_solve(p_solve)
    out["state"] = ctx.get_state()
    out["r_pde"] = ctx.residual()[1]
    st = ctx.iterate_to_tolerance(1, p_solve, 0.3 * out["r_pde"], 400)
    out["iters"] = st.iterations
    res, recs = run_ctx.run(sched)
    out["records"] = [(r.compliance, r.volume, r.unity, r.r_pde, r.separation, tuple(r.volume_fractions)[:2])
                      for r in recs]
    out["phases"] = run_ctx.get_phases(phases_buf)
    out["loops"] = (res.loops, res.termination)
    return out


kr = slab.slab_range(rank, nranks, g.n[axis])
ctx = D.Context(g, 1, 0.3, mode, k_range=kr, x_outermost=xo)
setup_solver(ctx)
join(ctx)
rc = D.Context.from_problem(prob, mode, k_range=kr, x_outermost=xo)
join(rc)
mine = work(ctx, rc, np.full(prob.nphases * N, np.nan))
outs = [None] * nranks
dist.all_gather_object(outs, mine)
if rank == 0:
    one = D.Context(g, 1, 0.3, mode, x_outermost=xo)
    setup_solver(one)
    ref = work(one, D.Context.from_problem(prob, mode, x_outermost=xo))
    cur = np.full(3 * N, np.nan)
    prev = np.full(3 * N, np.nan)
    phases = np.full(prob.nphases * N, np.nan)
    nd = np.array(g.n)
    idx = np.arange(N).reshape(nd[2], nd[1], nd[0])  # host x-fastest: [k][j][i]
    for r, o in enumerate(outs):
        a, b = slab.slab_range(r, nranks, g.n[axis])
        sl = (idx[:, :, a:b] if xo else idx[a:b]).ravel()
        c, p = o["state"]
        for comp in range(3):
            cur[comp * N + sl] = c[comp * N + sl]
            prev[comp * N + sl] = p[comp * N + sl]
        for q in range(prob.nphases):
            phases[q * N + sl] = o["phases"][q * N + sl]
    res = {
        "ok": True, "nranks": nranks, "mode": sys.argv[1], "layout": sys.argv[2], "halo": halo,
        "state_max_rel": float(np.abs(cur - ref["state"][0]).max() / np.abs(ref["state"][0]).max()),
        "state_bit_identical": bool(np.array_equal(cur, ref["state"][0]) and np.array_equal(prev, ref["state"][1])),
        "r_pde": [outs[0]["r_pde"], ref["r_pde"]],
        "iters": [outs[0]["iters"], ref["iters"]],
        "records_same_on_all_ranks": all(o["records"] == outs[0]["records"] for o in outs),
        "records_bit_identical": outs[0]["records"] == ref["records"],
        "records_max_rel": max(abs(x - y) / max(abs(y), 1e-300) for ra, rb in zip(outs[0]["records"], ref["records"])
                               for x, y in zip(ra[:5], rb[:5])) if outs[0]["records"] else float("inf"),
        "nrecords": [len(o["records"]) for o in outs] + [len(ref["records"])],
        "phases_max_abs": float(np.abs(phases - ref["phases"]).max()),
        "loops": [outs[0]["loops"], ref["loops"]],
    }
    print(json.dumps(res), flush=True)
dist.barrier()
dist.destroy_process_group()

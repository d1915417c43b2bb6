"""TEST INFRASTRUCTURE: the NCCL path of the slab decomposition with several ranks
on one GPU, through the in-process NCCL emulator (tests/nccl_emu/nccl_emu.cu).

    CUDA_DEVICE_MAX_CONNECTIONS=32 CUDA_MODULE_LOADING=EAGER PETTO_NCCL_LIB=tests/nccl_emu/libnccl_emu.so \
        python tests/nccl_emu/run_ranks.py NRANKS replica|fast [x]

Every rank is a host thread with its own slab context and communicator
(petto_dev_comm_init) -- the code path of one process per GPU under torchrun --
and runs: hybrid_solve (NCCL ghost planes every step), the residual norm,
iterate_to_tolerance, and a 3-loop run() (phi/mu halos, all-reduced scalars,
REPLICA chained sums, node-0 broadcast).  Rank 0 prints one JSON line comparing
the gathered results with the single-domain context."""
import faulthandler
import json
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2509_06971_b200 import device as D  # noqa: E402
from paper_2509_06971_b200 import problem as P  # noqa: E402
from paper_2509_06971_b200 import slab  # noqa: E402

if os.environ.get("EMU_TRACE") == "1":
    faulthandler.dump_traceback_later(35, exit=True)  # where every thread is if a rank hangs
nranks = int(sys.argv[1])
mode = D.MODE_REPLICA if sys.argv[2] == "replica" else D.MODE_FAST
xo = len(sys.argv) > 3 and sys.argv[3] == "x"
cfg = P.config("C4", nx=40, ny=14, nz=13, n_apt=30, n_pt=30, max_loops=3, report_every=1)
prob = P.build_problem(cfg)
g = prob.grid
sched = P.build_schedule(cfg, g, spectral_bound=D.spectral_bound)
axis = 0 if xo else 2
rng = np.random.default_rng(5)
u0 = rng.uniform(-1e-3, 1e-3, 3 * g.num_nodes)
E = np.maximum(1e-6, rng.random(g.num_nodes) ** 3)
p_solve = P.PTParams(sched.pt.dt_pt, sched.pt.dt_apt, sched.pt.theta, 37, 11, sched.pt.form)


def setup_solver(ctx):
    ctx.set_constraints(prob.cons_entry, prob.cons_value)
    ctx.set_source(prob.source)
    ctx.set_property(E)
    ctx.init_operator()
    ctx.set_state(u0, u0)


TRACE = os.environ.get("EMU_TRACE") == "1"


def trace(*a):
    if TRACE:
        print(*a, file=sys.stderr, flush=True)


def work(ctx, run_ctx, out, tag=""):
    """The operation sequence every rank (and the single domain) runs."""
    trace(tag, "hybrid_solve")
    ctx.hybrid_solve(p_solve)
    out["state"] = ctx.get_state()
    trace(tag, "residual")
    out["r_pde"] = ctx.residual()[1]
    trace(tag, "iterate_to_tolerance")
    st = ctx.iterate_to_tolerance(1, p_solve, 0.3 * out["r_pde"], 400)
    out["iters"] = st.iterations
    out["r_final"] = st.r_final
    trace(tag, "run")
    res, recs = run_ctx.run(sched)
    trace(tag, "done")
    out["records"] = [(r.compliance, r.volume, r.unity, r.r_pde, r.separation, tuple(r.volume_fractions)[:2])
                      for r in recs]
    out["phases"] = run_ctx.get_phases(out.get("phases_buf"))
    out["loops"] = (res.loops, res.termination)


# the single domain
one = D.Context(g, 1, 0.3, mode, x_outermost=xo)
setup_solver(one)
ref = {}
work(one, D.Context.from_problem(prob, mode, x_outermost=xo), ref, "single")
del one  # fewer streams: each needs a hardware work queue of its own (nccl_emu.cu)

uid = D.comm_unique_id()
outs = [dict() for _ in range(nranks)]
errs = []
N = g.num_nodes


def rank_main(r):
    try:
        kr = slab.slab_range(r, nranks, g.n[axis])
        ctx = D.Context(g, 1, 0.3, mode, k_range=kr, x_outermost=xo)
        setup_solver(ctx)
        trace(r, "comm_init")
        ctx.comm_init(uid, r, nranks)
        rc = D.Context.from_problem(prob, mode, k_range=kr, x_outermost=xo)
        rc.comm_init(uid2, r, nranks)  # the run() contexts' own communicator
        outs[r]["phases_buf"] = phases_all
        trace(r, "ready")
        work(ctx, rc, outs[r], r)
    except Exception as ex:  # noqa: BLE001
        errs.append(f"rank {r}: {ex!r}")


uid2 = D.comm_unique_id()  # the run() contexts' communicator
phases_all = np.full(prob.nphases * N, np.nan)
th = [threading.Thread(target=rank_main, args=(r,)) for r in range(nranks)]
for t in th:
    t.start()
for t in th:
    t.join()
if errs:
    print(json.dumps({"ok": False, "errors": errs}))
    sys.exit(1)
cur = np.full(3 * N, np.nan)
prev = np.full(3 * N, np.nan)
# each rank's get_state filled only its owned planes of its own arrays: merge them
kr = [slab.slab_range(r, nranks, g.n[axis]) for r in range(nranks)]
nd = np.array(g.n)
for r, o in enumerate(outs):
    c, p = o["state"]
    idx = np.arange(N).reshape(nd[2], nd[1], nd[0])  # host x-fastest: [k][j][i]
    sl = idx[:, :, kr[r][0]:kr[r][1]] if xo else idx[kr[r][0]:kr[r][1]]
    sl = sl.ravel()
    for comp in range(3):
        cur[comp * N + sl] = c[comp * N + sl]
        prev[comp * N + sl] = p[comp * N + sl]
rec_ok = all(o["records"] == outs[0]["records"] for o in outs)
res = {
    "ok": True, "nranks": nranks, "mode": sys.argv[2], "layout": "x" if xo else "z",
    "state_max_rel": float(np.abs(cur - ref["state"][0]).max() / np.abs(ref["state"][0]).max()),
    "prev_max_rel": float(np.abs(prev - ref["state"][1]).max() / np.abs(ref["state"][1]).max()),
    "state_bit_identical": bool(np.array_equal(cur, ref["state"][0]) and np.array_equal(prev, ref["state"][1])),
    "r_pde": [outs[0]["r_pde"], ref["r_pde"]],
    "iters": [outs[0]["iters"], ref["iters"]],
    "records_same_on_all_ranks": rec_ok,
    "records_bit_identical": outs[0]["records"] == ref["records"],
    "records_max_rel": max(abs(a - b) / max(abs(b), 1e-300) for ra, rb in zip(outs[0]["records"], ref["records"])
                           for a, b in zip(ra[:5], rb[:5])),
    "phases_max_abs": float(np.abs(phases_all - ref["phases"]).max()),
    "loops": [outs[0]["loops"], ref["loops"]],
}
print(json.dumps(res))

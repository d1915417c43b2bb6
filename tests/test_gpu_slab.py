"""GPU: the slab decomposition on one B200 (a local group of contexts, one per
slab, exchanging ghost planes by stream-ordered copies).  Each node's update does
not depend on how the z axis is split, so the group must reproduce the
single-domain fused solve bit for bit."""
import numpy as np
import pytest

from paper_2509_06971_b200 import device as D
from paper_2509_06971_b200 import problem as P
from paper_2509_06971_b200 import slab

from . import helpers as H

pytestmark = pytest.mark.gpu


def inputs(g, physics):
    comps = g.dim if physics else 1
    prop = H.random_modulus(g, 5) if physics else H.rng(4).uniform(0.5, 2.0, g.num_nodes)
    src = H.sparse_loads(g, comps, 2) if physics else np.full(g.num_nodes, 0.3)
    bc = H.elastic_bc(g, "x_hi") if physics else H.heat_bc(g, ("x_lo", "z_hi"))
    cur = H.random_field(comps * g.num_nodes, 1, -0.01, 0.01)
    prev = H.random_field(comps * g.num_nodes, 2, -0.01, 0.01)
    return comps, prop, src, bc, cur, prev


@pytest.mark.parametrize("physics", [1, 0])
@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("mode", [D.MODE_FAST, D.MODE_REPLICA])
def test_group_equals_single_domain(physics, nranks, mode):
    g = P.Grid.make3d(40, 17, 14, 2.0, 1.0, 0.7)
    comps, prop, src, bc, cur, prev = inputs(g, physics)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=23, n_pt=9, form=1)
    e, v = P.make_constraints(g, bc, comps)

    def setup(ctx):
        ctx.set_constraints(e, v)
        ctx.set_source(src)
        ctx.set_property(prop)
        ctx.init_operator()
        ctx.set_state(cur, prev)

    one = D.Context(g, physics, 0.3, mode)
    setup(one)
    one.hybrid_solve(p)
    want_c, want_p = one.get_state()

    ctxs = [D.Context(g, physics, 0.3, mode, k_range=slab.slab_range(r, nranks, g.n[2])) for r in range(nranks)]
    for c in ctxs:
        setup(c)
    D.group_link(ctxs)
    D.group_hybrid_solve(ctxs, p)
    got_c = np.full(comps * g.num_nodes, np.nan)
    got_p = np.full(comps * g.num_nodes, np.nan)
    for c in ctxs:
        c.get_state(got_c, got_p)  # each fills its owned planes
    assert np.array_equal(got_c, want_c) and np.array_equal(got_p, want_p)


@pytest.mark.parametrize("mode", [D.MODE_FAST, D.MODE_REPLICA])
def test_single_rank_nccl_paths(mode):
    """A one-rank NCCL communicator runs the distributed code paths (halo no-ops,
    all-reduced norms, device-side stop test after the all-reduce) and must give
    the same answers as the plain context."""
    g = P.Grid.make3d(33, 12, 10, 2.0, 1.0, 0.7)
    comps, prop, src, bc, cur, prev = inputs(g, 1)
    e, v = P.make_constraints(g, bc, comps)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.2 * h, theta=1.0, n_apt=30, n_pt=10, form=1)
    outs = []
    for use_comm in (False, True):
        ctx = D.Context(g, 1, 0.3, mode)
        ctx.set_constraints(e, v)
        ctx.set_source(src)
        ctx.set_property(prop)
        ctx.init_operator()
        if use_comm:
            ctx.comm_init(D.comm_unique_id(), 0, 1)
        ctx.set_state(cur, prev)
        ctx.hybrid_solve(p)
        r, rp = ctx.residual()
        st = ctx.iterate_to_tolerance(1, p, 0.5 * rp, 500)
        outs.append((ctx.get_state()[0], r, rp, st.iterations, st.r_final))
    a, b = outs
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert a[2] == b[2] and a[3] == b[3] and a[4] == b[4]


def test_group_c4_size_fast():
    """C4 geometry split in 4 slabs: 50 semi-implicit APT steps, bit-identical."""
    cfg = P.config("C4")
    prob = P.build_problem(cfg)
    g = prob.grid
    E = H.random_modulus(g, 3)
    sched = P.build_schedule(cfg, g, spectral_bound=D.spectral_bound)
    p = P.PTParams(sched.pt.dt_pt, sched.pt.dt_apt, 1.0, 50, 0, 1)
    state = H.random_field(3 * g.num_nodes, 4, -1e-3, 1e-3)

    def setup(ctx):
        ctx.set_constraints(prob.cons_entry, prob.cons_value)
        ctx.set_source(prob.source)
        ctx.set_property(E)
        ctx.init_operator()
        ctx.set_state(state, state)

    one = D.Context(g, 1, 0.3)
    setup(one)
    one.hybrid_solve(p)
    want, _ = one.get_state()
    ctxs = [D.Context(g, 1, 0.3, k_range=slab.slab_range(r, 4, g.n[2])) for r in range(4)]
    for c in ctxs:
        setup(c)
    D.group_link(ctxs)
    D.group_hybrid_solve(ctxs, p)
    got = np.full(3 * g.num_nodes, np.nan)
    for c in ctxs:
        c.get_state(got, np.zeros(3 * g.num_nodes))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("nranks", [2, 3])
def test_group_repeated_solves_with_new_states(nranks):
    """Peer halo across solves: the state upload between two group solves is a
    step of the neighbour protocol (no stale or overwritten ghost planes)."""
    g = P.Grid.make3d(36, 16, 13, 2.0, 1.0, 0.7)
    comps, prop, src, bc, cur, prev = inputs(g, 1)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=17, n_pt=4, form=1)
    e, v = P.make_constraints(g, bc, comps)
    cur2 = H.random_field(comps * g.num_nodes, 11, -0.02, 0.02)

    def setup(ctx):
        ctx.set_constraints(e, v)
        ctx.set_source(src)
        ctx.set_property(prop)
        ctx.init_operator()
        ctx.set_state(cur, prev)

    one = D.Context(g, 1, 0.3)
    setup(one)
    one.hybrid_solve(p)
    one.set_state(cur2, cur)
    one.hybrid_solve(p)
    want_c, want_p = one.get_state()

    ctxs = [D.Context(g, 1, 0.3, k_range=slab.slab_range(r, nranks, g.n[2])) for r in range(nranks)]
    for c in ctxs:
        setup(c)
    D.group_link(ctxs)
    D.group_hybrid_solve(ctxs, p)
    for c in ctxs:
        c.set_state(cur2, cur)
    D.group_hybrid_solve(ctxs, p)
    got_c = np.full(comps * g.num_nodes, np.nan)
    got_p = np.full(comps * g.num_nodes, np.nan)
    for c in ctxs:
        c.get_state(got_c, got_p)
    assert np.array_equal(got_c, want_c) and np.array_equal(got_p, want_p)


@pytest.mark.parametrize("nproc", [2, 3])
def test_peer_halo_multiprocess(nproc):
    """Peer halo across processes (CUDA IPC + cross-process stream flags): ranks
    share the one GPU; only streams wait on flags, no kernel waits on a rank."""
    import os
    import socket
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.join(root, "tools", "mp_peer_check.py"), "--device", "0"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert f"peer halo, {nproc} processes: bit-identical" in r.stdout


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



# --------------------------------------------------------------- design loop
# The whole run() on slabs: ghost planes of phi and mu around the
# Cahn-Hilliard kernels, every global scalar reduced over the slabs (REPLICA: one
# serial sum chained across the slabs in order), node 0's Lame pair shared.


def _slabs(prob, nranks, mode):
    ctxs = [D.Context.from_problem(prob, mode, k_range=slab.slab_range(r, nranks, prob.grid.n[2]))
            for r in range(nranks)]
    D.group_link(ctxs)
    return ctxs


def _gather_phases(ctxs, prob):
    out = np.full(prob.nphases * prob.grid.num_nodes, np.nan)
    for c in ctxs:
        c.get_phases(out)
    return out


RUN_SLAB_CASES = [
    ("C4", dict(max_loops=3, report_every=1), [2, 3, 4]),                      # full C4 grid, 3 loops
    ("drone3d", dict(nx=24, ny=12, nz=20, n_apt=20, n_pt=20, max_loops=3, report_every=1), [3]),  # heat + region
]


def _config(name, kw):
    if name in P.CONFIGS:
        return P.config(name, **kw)
    cfg = P.make_preset(name)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


@pytest.mark.parametrize("mode", [D.MODE_REPLICA, D.MODE_FAST])
@pytest.mark.parametrize("case", range(len(RUN_SLAB_CASES)))
def test_group_run_equals_single_domain(case, mode):
    name, kw, splits = RUN_SLAB_CASES[case]
    cfg = _config(name, kw)
    prob = P.build_problem(cfg)
    sched = P.build_schedule(cfg, prob.grid, spectral_bound=D.spectral_bound)
    one = D.Context.from_problem(prob, mode)
    wres, wrecs = one.run(sched)
    wph = one.get_phases()
    wst = one.get_state()[0]
    for nranks in splits:
        ctxs = _slabs(prob, nranks, mode)
        res, recs = D.group_run(ctxs, sched)
        assert (res.loops, res.termination, res.apt_steps, res.pt_steps) == (
            wres.loops, wres.termination, wres.apt_steps, wres.pt_steps)
        ph = _gather_phases(ctxs, prob)
        st = np.full(prob.comps * prob.grid.num_nodes, np.nan)
        for c in ctxs:
            c.get_state(st, None)
        fields = ("compliance", "volume", "unity", "region", "r_pde", "separation")
        if mode == D.MODE_REPLICA:
            for a, b in zip(recs, wrecs):
                assert [getattr(a, f) for f in fields] == [getattr(b, f) for f in fields]
                assert list(a.volume_fractions) == list(b.volume_fractions)
            assert np.array_equal(ph, wph) and np.array_equal(st, wst)
            assert res.clamp_mass_drift == wres.clamp_mass_drift
        else:
            for a, b in zip(recs, wrecs):
                for f in fields:
                    x, y = getattr(a, f), getattr(b, f)
                    assert abs(x - y) <= 1e-12 * max(abs(y), 1e-30), (nranks, f, x, y)
            assert np.abs(ph - wph).max() <= 1e-12
            assert np.abs(st - wst).max() <= 1e-12 * np.abs(wst).max()
        del ctxs


@pytest.mark.parametrize("nranks", [2, 3])
def test_group_design_calls_replica_bit_exact(nranks):
    """design_update, ch_step, objectives and the residual norm of a split grid,
    call by call, bit-identical to one domain (REPLICA)."""
    cfg = P.config("C4", nx=40, ny=17, nz=14)
    prob = P.build_problem(cfg)
    g = prob.grid
    sched = P.build_schedule(cfg, g, spectral_bound=D.spectral_bound)
    state = H.random_field(3 * g.num_nodes, 8, -0.15, 0.15)
    phases = H.rng(42).uniform(0.2, 0.8, prob.nphases * g.num_nodes)
    one = D.Context.from_problem(prob, D.MODE_REPLICA)
    ctxs = _slabs(prob, nranks, D.MODE_REPLICA)
    for c in [one] + ctxs:
        c.set_phases(phases)
        c.set_state(state, state)
    one.interpolate(download=False)
    one.init_operator()
    D.group_interpolate(ctxs)
    D.group_init_operator(ctxs)
    assert D.group_residual(ctxs) == one.residual()[1]
    rep1, sep1 = one.objectives()
    rep2, sep2 = D.group_objectives(ctxs)
    assert (rep1.compliance, rep1.unity, rep1.volume, sep1) == (rep2.compliance, rep2.unity, rep2.volume, sep2)
    one.design_update()
    D.group_design_update(ctxs)
    assert np.array_equal(_gather_phases(ctxs, prob), one.get_phases())
    s1 = one.ch_step(sched.ch_mobility, sched.ch_gamma, sched.dt_ch)
    s2 = D.group_ch_step(ctxs, sched.ch_mobility, sched.ch_gamma, sched.dt_ch)
    assert s1 == s2
    assert np.array_equal(_gather_phases(ctxs, prob), one.get_phases())


def test_linked_slab_refuses_single_context_calls():
    """A slab of a local group has no collectives of its own: the single-context
    design / run / residual entry points refuse it instead of computing slab-local
    sums (the group entry points are the way in)."""
    cfg = P.config("C4", nx=24, ny=10, nz=12)
    prob = P.build_problem(cfg)
    sched = P.build_schedule(cfg, prob.grid, spectral_bound=D.spectral_bound)
    ctxs = _slabs(prob, 2, D.MODE_FAST)
    for call in (lambda c: c.run(sched), lambda c: c.design_update(), lambda c: c.objectives(),
                 lambda c: c.ch_step(1.0, 3e-5, 1e-6), lambda c: c.residual()):
        with pytest.raises(ValueError, match="group"):
            call(ctxs[1])
    lone = D.Context.from_problem(prob, D.MODE_FAST, k_range=(0, 6))  # a slab without a communicator
    with pytest.raises(ValueError, match="communicator"):
        lone.run(sched)


@pytest.mark.parametrize("mode", [D.MODE_FAST, D.MODE_REPLICA])
def test_group_abort_at_same_check_as_single_domain(mode):
    """A non-finite value on the first slab spreads one plane per step and reaches
    the last slab only after the first check_finite (step 100).  Every slab learns
    the first non-finite step of any slab at each check, so all stop at step 100
    like the single domain (without that reduction the last slab would run on to
    step 200) and the state left behind is the single domain's state."""
    g = P.Grid.make3d(16, 8, 240, 1.0, 0.5, 15.0)
    comps, prop, src, bc, cur, prev = inputs(g, 1)
    cur = cur.copy()
    cur[g.node(0, 4, 2)] = np.nan
    e, v = P.make_constraints(g, bc, comps)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=0, n_pt=450, form=1)

    def setup(ctx):
        ctx.set_constraints(e, v)
        ctx.set_source(src)
        ctx.set_property(prop)
        ctx.init_operator()
        ctx.set_state(cur, prev)

    one = D.Context(g, 1, 0.3, mode)
    setup(one)
    with pytest.raises(D.NumericalAbort) as ex1:
        one.hybrid_solve(p)
    want = one.get_state()[0]
    ctxs = [D.Context(g, 1, 0.3, mode, k_range=slab.slab_range(r, 3, g.n[2])) for r in range(3)]
    for c in ctxs:
        setup(c)
    D.group_link(ctxs)
    with pytest.raises(D.NumericalAbort) as ex2:
        D.group_hybrid_solve(ctxs, p)
    assert ex1.value.step == ex2.value.step == 100
    got = np.full(comps * g.num_nodes, np.nan)
    for c in ctxs:
        c.get_state(got, None)
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin) and 0 < fin.sum() < fin.size
    assert np.array_equal(got[fin], want[fin])


@pytest.mark.parametrize("mode", [D.MODE_REPLICA, D.MODE_FAST])
@pytest.mark.parametrize("nranks", [2, 3])
def test_group_iterate_to_tolerance(nranks, mode):
    """iterate_to_tolerance (state_solver.hpp:511-541) on slabs: r^2 reduced over the
    slabs every step (REPLICA chained: the same iteration count and state bit for
    bit), the new state's ghost planes exchanged before the next step."""
    g = P.Grid.make3d(33, 12, 14, 2.0, 1.0, 0.7)
    comps, prop, src, bc, cur, prev = inputs(g, 1)
    e, v = P.make_constraints(g, bc, comps)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.2 * h, theta=1.0, n_apt=30, n_pt=10, form=1)

    def setup(ctx):
        ctx.set_constraints(e, v)
        ctx.set_source(src)
        ctx.set_property(prop)
        ctx.init_operator()
        ctx.set_state(cur, prev)

    one = D.Context(g, 1, 0.3, mode)
    setup(one)
    r0 = one.residual()[1]
    setup(one)
    want = one.iterate_to_tolerance(1, p, 0.2 * r0, 3000)
    want_u = one.get_state()[0]
    ctxs = [D.Context(g, 1, 0.3, mode, k_range=slab.slab_range(r, nranks, g.n[2])) for r in range(nranks)]
    for c in ctxs:
        setup(c)
    D.group_link(ctxs)
    got = D.group_iterate_to_tolerance(ctxs, 1, p, 0.2 * r0, 3000)
    got_u = np.full(comps * g.num_nodes, np.nan)
    for c in ctxs:
        c.get_state(got_u, None)
    assert got.converged == want.converged
    if mode == D.MODE_REPLICA:
        assert (got.iterations, got.r_initial, got.r_final) == (want.iterations, want.r_initial, want.r_final)
        assert np.array_equal(got_u, want_u)
    else:
        assert abs(got.iterations - want.iterations) <= 1
        assert abs(got.r_initial - want.r_initial) <= 1e-13 * want.r_initial

"""GPU: the x-outermost device layout (petto_grid_desc.x_outermost) and slabs along
x, the longest axis of the cantilever configs.  The device keeps
the grid as (y, z, x) with the displacement components permuted alike; uploads
and downloads permute, so callers keep the reference's x-fastest arrays.  The
operator is an axis relabelling of an isotropic one: FAST results agree with the
reference layout to rounding (1e-12 per residual, 1e-10 per solve), and a split
along x is bit-identical to the unsplit permuted grid for the state solve."""
import numpy as np
import pytest

from paper_2509_06971_b200 import device as D
from paper_2509_06971_b200 import problem as P
from paper_2509_06971_b200 import slab

from . import helpers as H

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


GRIDS = [P.Grid.make3d(40, 17, 12, 2.0, 1.0, 0.7), P.Grid.make3d(70, 23, 19, 2.0, 1.0, 1.0)]


def elastic_setup(g, ctx, seed=0):
    E = H.random_modulus(g, 3 + seed)
    f = H.sparse_loads(g, 3, 5 + seed, count=30)
    bc = H.elastic_bc(g, "x_hi", pins=[(g.node(0, 0, 0), 1, 0.01), (g.node(3, 2, 1), 2, -0.02)])
    bc.face[P.FACE_NAMES.index("z_lo")] = P.FaceCondition(P.ROLLER, 0.0, 2)  # a roller: one pinned component
    e, v = P.make_constraints(g, bc, 3)
    ctx.set_constraints(e, v)
    ctx.set_source(f)
    ctx.set_property(E)
    ctx.init_operator()


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_upload_download_round_trip(gi):
    g = GRIDS[gi]
    u = H.random_field(3 * g.num_nodes, 1)
    w = H.random_field(3 * g.num_nodes, 2)
    ctx = D.Context(g, 1, 0.3, x_outermost=True)
    ctx.set_state(u, w)
    c, p = ctx.get_state()
    assert np.array_equal(c, u) and np.array_equal(p, w)


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_elastic_residual_and_solve_match_reference_layout(gi):
    g = GRIDS[gi]
    u = H.random_field(3 * g.num_nodes, 7, -0.01, 0.01)
    up = H.random_field(3 * g.num_nodes, 8, -0.01, 0.01)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=50, n_pt=10, form=1)
    outs = []
    for perm in (False, True):
        ctx = D.Context(g, 1, 0.3, x_outermost=perm)
        elastic_setup(g, ctx)
        ctx.set_state(u, up)
        r, rn = ctx.residual()
        ctx.hybrid_solve(p)
        outs.append((r, rn, ctx.get_state()))
    (r0, n0, s0), (r1, n1, s1) = outs
    assert rel(r1, r0) < 1e-12 and abs(n1 - n0) <= 1e-12 * n0
    assert rel(s1[0], s0[0]) < 1e-10 and rel(s1[1], s0[1]) < 1e-10


def test_heat_solve_matches_reference_layout():
    g = GRIDS[1]
    kappa = H.rng(4).uniform(0.5, 2.0, g.num_nodes)
    src = H.rng(5).uniform(0.0, 1.0, g.num_nodes)
    bc = H.heat_bc(g, ("x_lo", "z_hi"), 0.25)
    e, v = P.make_constraints(g, bc, 1)
    T = H.random_field(g.num_nodes, 3, 0.0, 0.1)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.2 * h, theta=1.0, n_apt=40, n_pt=20, form=0)
    outs = []
    for perm in (False, True):
        ctx = D.Context(g, 0, 0.3, x_outermost=perm)
        ctx.set_constraints(e, v)
        ctx.set_source(src)
        ctx.set_property(kappa)
        ctx.init_operator()
        ctx.set_state(T, T)
        ctx.hybrid_solve(p)
        outs.append(ctx.get_state()[0])
    assert rel(outs[1], outs[0]) < 1e-12


RUN_CASES = [
    ("C4", dict(nx=40, ny=14, nz=12, n_apt=40, n_pt=40, max_loops=3, report_every=1)),
    ("drone3d", dict(nx=24, ny=12, nz=20, n_apt=20, n_pt=20, max_loops=3, report_every=1)),
]


def _config(name, kw):
    if name in P.CONFIGS:
        return P.config(name, **kw)
    cfg = P.make_preset(name)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


@pytest.mark.parametrize("case", range(len(RUN_CASES)))
def test_run_matches_reference_layout_and_x_slabs(case):
    """run() on the permuted grid vs the reference layout (rounding only), and on
    2 / 3 slabs along x vs the unsplit permuted grid."""
    name, kw = RUN_CASES[case]
    cfg = _config(name, kw)
    prob = P.build_problem(cfg)
    sched = P.build_schedule(cfg, prob.grid, spectral_bound=D.spectral_bound)
    ref = D.Context.from_problem(prob)
    wres, wrecs = ref.run(sched)
    perm = D.Context.from_problem(prob, x_outermost=True)
    pres, precs = perm.run(sched)
    fields = ("compliance", "volume", "unity", "region", "r_pde")
    assert (pres.loops, pres.termination) == (wres.loops, wres.termination)
    for a, b in zip(precs, wrecs):
        for f in fields:
            x, y = getattr(a, f), getattr(b, f)
            assert abs(x - y) <= 1e-10 * max(abs(y), 1e-30), (f, x, y)
        assert a.separation == b.separation
    assert np.abs(perm.get_phases() - ref.get_phases()).max() < 1e-10
    for nranks in (2, 3):
        ctxs = [D.Context.from_problem(prob, k_range=slab.slab_range(r, nranks, prob.grid.n[0]), x_outermost=True)
                for r in range(nranks)]
        D.group_link(ctxs)
        res, recs = D.group_run(ctxs, sched)
        assert (res.loops, res.termination) == (pres.loops, pres.termination)
        for a, b in zip(recs, precs):
            for f in fields:
                x, y = getattr(a, f), getattr(b, f)
                assert abs(x - y) <= 1e-12 * max(abs(y), 1e-30), (nranks, f, x, y)
        ph = np.full(prob.nphases * prob.grid.num_nodes, np.nan)
        for c in ctxs:
            c.get_phases(ph)
        assert np.abs(ph - perm.get_phases()).max() <= 1e-12


@pytest.mark.parametrize("nranks", [2, 4])
def test_x_slab_group_solve_bit_identical(nranks):
    g = GRIDS[1]
    u = H.random_field(3 * g.num_nodes, 7, -0.01, 0.01)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=30, n_pt=7, form=1)
    one = D.Context(g, 1, 0.3, x_outermost=True)
    elastic_setup(g, one)
    one.set_state(u, u)
    one.hybrid_solve(p)
    want = one.get_state()
    ctxs = [D.Context(g, 1, 0.3, k_range=slab.slab_range(r, nranks, g.n[0]), x_outermost=True) for r in range(nranks)]
    for c in ctxs:
        elastic_setup(g, c)
        c.set_state(u, u)
    D.group_link(ctxs)
    D.group_hybrid_solve(ctxs, p)
    got_c = np.full(3 * g.num_nodes, np.nan)
    got_p = np.full(3 * g.num_nodes, np.nan)
    for c in ctxs:
        c.get_state(got_c, got_p)
    assert np.array_equal(got_c, want[0]) and np.array_equal(got_p, want[1])


def test_x_outermost_refuses_replica_and_writers(tmp_path):
    g = GRIDS[0]
    with pytest.raises(ValueError, match="FAST"):
        D.Context(g, 1, 0.3, mode=D.MODE_REPLICA, x_outermost=True)
    ctx = D.Context(g, 1, 0.3, x_outermost=True)
    with pytest.raises(ValueError, match="FAST"):
        ctx.set_mode(D.MODE_REPLICA)
    ctx.set_state(np.zeros(3 * g.num_nodes))
    with pytest.raises(ValueError, match="reference layout"):
        ctx.write_field_csv(0, 0, tmp_path / "u.csv")

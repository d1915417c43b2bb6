"""GPU parity of the state path through the C-ABI.

REPLICA mode must be bit-identical to the oracle (which is pinned bitwise to the
reference in test_oracle_port.py).  FAST mode (the fused sm_100a kernels) must
agree to 1e-12 relative per residual / step and 1e-10 after a few hundred steps
(SURVEY.md 8c "fast mode" tolerances).
"""
import numpy as np
import pytest

from paper_2509_06971_b200 import device as D
from paper_2509_06971_b200 import problem as P

from . import helpers as H

pytestmark = pytest.mark.gpu

FAST, REPLICA = D.MODE_FAST, D.MODE_REPLICA


def rel_err(a, b):
    scale = max(np.abs(b).max(), 1e-300)
    return float(np.abs(a - b).max() / scale)


ELASTIC_GRIDS = [
    P.Grid.make2d(17, 9, 2.0, 1.0),
    P.Grid.make2d(33, 20, 4.0, 1.0),
    P.Grid.make3d(7, 6, 5, 1.0, 0.8, 0.6),
    P.Grid.make3d(12, 9, 10, 2.0, 1.0, 1.0),
    P.Grid.make3d(37, 15, 11, 2.0, 1.0, 0.7),   # nx > 32, ragged tiles
    P.Grid.make3d(70, 23, 19, 2.0, 1.0, 1.0),   # several x tiles and strips
]


def elastic_case(g, seed):
    d = g.dim
    E = H.random_modulus(g, seed=seed + 1)
    u = H.random_field(d * g.num_nodes, seed=7 + seed)
    up = H.random_field(d * g.num_nodes, seed=17 + seed)
    f = H.sparse_loads(g, d, seed=3 + seed)
    bc = H.elastic_bc(g, "x_hi", pins=[(g.node(0, 0), 1, 0.0), (g.node(1, 2), 0, 0.25)])
    return E, u, up, f, bc


@pytest.mark.parametrize("gi", range(len(ELASTIC_GRIDS)))
@pytest.mark.parametrize("mode", [REPLICA, FAST])
def test_elasticity_residual(port, gi, mode):
    g = ELASTIC_GRIDS[gi]
    E, u, _, f, bc = elastic_case(g, gi)
    want = port.elasticity_residual(g, bc, E, 0.3, f, u)
    op = D.ElasticityOperator(g, E, 0.3, f, bc, mode=mode)
    got = op.residual(u)
    if mode == REPLICA:
        assert np.array_equal(got, want)
    else:
        assert rel_err(got, want) < 1e-12


HEAT_GRIDS = [P.Grid.make2d(16, 16, 4.0, 4.0), P.Grid.make2d(45, 31, 1.0, 1.0), P.Grid.make3d(9, 8, 7, 1.0, 1.0, 1.0)]


@pytest.mark.parametrize("gi", range(len(HEAT_GRIDS)))
@pytest.mark.parametrize("mode", [REPLICA, FAST])
@pytest.mark.parametrize("uniform", [True, False])
def test_heat_residual(port, gi, mode, uniform):
    g = HEAT_GRIDS[gi]
    kappa = H.rng(gi).uniform(0.5, 2.0, g.num_nodes)
    src = np.full(g.num_nodes, 0.01) if uniform else H.rng(gi + 9).uniform(-1, 1, g.num_nodes)
    T = H.random_field(g.num_nodes, 11 + gi, -1, 1)
    bc = H.heat_bc(g)
    want = port.heat_residual(g, bc, kappa, src, T)
    got = D.HeatOperator(g, kappa, src, bc, mode=mode).residual(T)
    if mode == REPLICA:
        assert np.array_equal(got, want)
    else:
        assert rel_err(got, want) < 1e-12


def test_heat_residual_known_answer():
    """tests/test_state_solver.cpp:51-61: 0.01 at free nodes, 0 at pinned."""
    g = P.Grid.make2d(16, 16, 4.0, 4.0)
    bc = P.BoundarySpec.all_faces(2, P.DIRICHLET)
    for mode in (REPLICA, FAST):
        r = D.HeatOperator(g, np.ones(g.num_nodes), np.full(g.num_nodes, 0.01), bc, mode=mode).residual(
            np.zeros(g.num_nodes))
        pinned = np.zeros(g.num_nodes, bool)
        pinned[P.make_constraints(g, bc, 1)[0]] = True
        assert np.all(r[pinned] == 0.0) and np.all(r[~pinned] == 0.01)


def test_elasticity_zero_state_known_answer():
    """tests/test_state_solver.cpp:153-177: r = 0 without loads, -1 on y under f_y = 1."""
    g = P.Grid.make2d(17, 9, 2.0, 1.0)
    bc = H.elastic_bc(g, None, pins=[(g.node(0, 0), 1, 0.0)])
    for mode in (REPLICA, FAST):
        loads = np.zeros(2 * g.num_nodes)
        op = D.ElasticityOperator(g, np.ones(g.num_nodes), 0.3, loads, bc, mode=mode)
        assert np.all(op.residual(np.zeros(2 * g.num_nodes)) == 0.0)
        loads[g.num_nodes:] = 1.0
        op = D.ElasticityOperator(g, np.ones(g.num_nodes), 0.3, loads, bc, mode=mode)
        r = op.residual(np.zeros(2 * g.num_nodes))
        assert np.all(r[: g.num_nodes] == 0.0)
        want = np.full(g.num_nodes, -1.0)
        want[g.node(0, 0)] = 0.0
        assert np.array_equal(r[g.num_nodes:], want)


@pytest.mark.parametrize("dim", [2, 3])
def test_elasticity_annihilates_affine(dim):
    """tests/test_state_solver.cpp:187-217 on the fast kernels."""
    g = P.Grid.make2d(9, 7, 1.0, 0.8) if dim == 2 else P.Grid.make3d(7, 6, 5, 1.0, 0.8, 0.6)
    bc = H.elastic_bc(g, None, pins=[(0, 0, 0.0)])
    grad = [[0.3, -0.1, 0.05], [0.2, 0.4, -0.15], [0.1, 0.0, 0.25]]
    i, j, k = g.ijk()
    x, y, z = (g.spacing[0] * i, g.spacing[1] * j, g.spacing[2] * k)
    u = np.concatenate([0.7 + grad[c][0] * x + grad[c][1] * y + (grad[c][2] * z if dim == 3 else 0) for c in range(dim)])
    for mode in (REPLICA, FAST):
        r = D.ElasticityOperator(g, np.ones(g.num_nodes), 0.3, np.zeros(dim * g.num_nodes), bc, mode=mode).residual(u)
        r = r.reshape(dim, g.n[2], g.n[1], g.n[0])
        inner = r[:, 1:-1, 1:-1, 1:-1] if dim == 3 else r[:, :, 1:-1, 1:-1]
        assert np.abs(inner).max() < 1e-10


def test_nonpositive_lame_rejected():
    g = P.Grid.make2d(5, 5, 1.0, 1.0)
    E = np.ones(g.num_nodes)
    E[7] = 0.0
    with pytest.raises(ValueError, match="Lame fields must be positive"):
        D.ElasticityOperator(g, E, 0.3, np.zeros(2 * g.num_nodes), H.elastic_bc(g, None))


HYBRID_CASES = [
    (0, 0, P.Grid.make2d(20, 12, 1.0, 1.0)),
    (0, 1, P.Grid.make3d(9, 7, 6, 1.0, 0.8, 0.6)),
    (1, 1, P.Grid.make2d(33, 17, 2.0, 1.0)),
    (1, 0, P.Grid.make2d(20, 12, 1.0, 1.0)),
    (1, 1, P.Grid.make3d(9, 7, 6, 1.0, 0.8, 0.6)),
    (1, 1, P.Grid.make3d(40, 17, 12, 2.0, 1.0, 0.7)),
    (1, 0, P.Grid.make3d(40, 17, 12, 2.0, 1.0, 0.7)),
]


def hybrid_inputs(physics, g):
    comps = g.dim if physics else 1
    prop = H.random_modulus(g, 5) if physics else H.rng(4).uniform(0.5, 2.0, g.num_nodes)
    src = H.sparse_loads(g, comps, 2) if physics else np.full(g.num_nodes, 0.3)
    bc = H.elastic_bc(g, "x_lo") if physics else H.heat_bc(g)
    cur = H.random_field(comps * g.num_nodes, 1, -0.01, 0.01)
    prev = H.random_field(comps * g.num_nodes, 2, -0.01, 0.01)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=37, n_pt=23)
    return comps, prop, src, bc, cur, prev, p


@pytest.mark.parametrize("case", range(len(HYBRID_CASES)))
@pytest.mark.parametrize("mode", [REPLICA, FAST])
def test_hybrid_solve(port, case, mode):
    physics, form, g = HYBRID_CASES[case]
    comps, prop, src, bc, cur, prev, p = hybrid_inputs(physics, g)
    p.form = form
    rc, wc, wp, _ = port.hybrid_solve(physics, g, bc, prop, 0.3, src, cur, prev, p)
    assert rc == 0
    op = D.DeviceOperator(g, physics, prop, src, bc, mode=mode)
    hist = D.StateHistory(cur.copy(), prev.copy())
    D.hybrid_solve(hist, op, p)
    if mode == REPLICA:
        assert np.array_equal(hist.current, wc) and np.array_equal(hist.previous, wp)
    else:
        assert rel_err(hist.current, wc) < 1e-10 and rel_err(hist.previous, wp) < 1e-10


def test_hybrid_zero_apt_equals_plain_pt(port):
    """tests/test_state_solver.cpp:230-249: n_apt = 0 is 25 PT steps bit for bit."""
    g = P.Grid.make2d(16, 16, 1.0, 1.0)
    bc = P.BoundarySpec.all_faces(2, P.DIRICHLET)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 4, dt_apt=h / 2, theta=1.0, n_apt=0, n_pt=25)
    op = D.HeatOperator(g, np.ones(g.num_nodes), np.ones(g.num_nodes), bc, mode=REPLICA)
    hist = D.StateHistory.of(np.zeros(g.num_nodes))
    D.hybrid_solve(hist, op, p)
    _, wc, _, _ = port.hybrid_solve(0, g, bc, np.ones(g.num_nodes), 0.3, np.ones(g.num_nodes),
                                    np.zeros(g.num_nodes), np.zeros(g.num_nodes), p)
    assert np.array_equal(hist.current, wc)


@pytest.mark.parametrize("mode", [REPLICA, FAST])
def test_reckless_step_aborts_at_check(mode):
    """tests/test_state_solver.cpp:330-340: NumericalAbort at the first check (step 100)."""
    g = P.Grid.make2d(16, 16, 1.0, 1.0)
    bc = P.BoundarySpec.all_faces(2, P.DIRICHLET)
    p = P.PTParams(dt_pt=1e6, dt_apt=0.5 / 15, theta=1.0, n_apt=0, n_pt=5000)
    op = D.HeatOperator(g, np.ones(g.num_nodes), np.ones(g.num_nodes), bc, mode=mode)
    hist = D.StateHistory.of(np.zeros(g.num_nodes))
    with pytest.raises(D.NumericalAbort) as ei:
        D.hybrid_solve(hist, op, p)
    assert ei.value.step == 100


@pytest.mark.parametrize("mode", [REPLICA, FAST])
def test_constrained_entries_exact_every_step(mode):
    """tests/test_state_solver.cpp:305-328: pinned entries stay bit-exact."""
    g = P.Grid.make2d(16, 12, 1.0, 1.0)
    bc = P.BoundarySpec()
    bc.face[0] = P.FaceCondition(P.DIRICHLET, 1.25, 0)
    bc.face[1] = P.FaceCondition(P.NEUMANN_ZERO, 0.0, 0)
    bc.face[2] = P.FaceCondition(P.DIRICHLET, -0.5, 0)
    bc.face[3] = P.FaceCondition(P.NEUMANN_ZERO, 0.0, 0)
    e, v = P.make_constraints(g, bc, 1)
    op = D.HeatOperator(g, np.ones(g.num_nodes), np.full(g.num_nodes, 0.3), bc, mode=mode)
    h = g.min_spacing()
    T = np.zeros(g.num_nodes)
    T[e] = v
    hist = D.StateHistory.of(T)
    for s in range(10):
        p = P.PTParams(dt_pt=h * h / 4, dt_apt=h / 2, theta=1.0, n_apt=s % 2, n_pt=1 - s % 2)
        D.hybrid_solve(hist, op, p)
        assert np.array_equal(hist.current[e], v)


@pytest.mark.parametrize("mode", [REPLICA, FAST])
@pytest.mark.parametrize("it_mode", [0, 1])
def test_iterate_to_tolerance_counts(port, mode, it_mode):
    g = P.Grid.make2d(24, 24, 1.0, 1.0)
    bc = P.BoundarySpec.all_faces(2, P.DIRICHLET)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 4, dt_apt=h / 2, theta=1.0, form=0)
    z = np.zeros(g.num_nodes)
    one = np.ones(g.num_nodes)
    rc, want, wc, wp = port.iterate_to_tolerance(0, g, bc, one, 0.3, one, z, z, it_mode, p, 1e-6, 100000)
    op = D.HeatOperator(g, one, one, bc, mode=mode)
    hist = D.StateHistory.of(z)
    got = D.iterate_to_tolerance(hist, op, it_mode, p, 1e-6, 100000)
    assert got.converged and want.converged
    if mode == REPLICA:
        assert got.iterations == want.iterations and got.r_final == want.r_final
        assert got.r_initial == want.r_initial
        assert np.array_equal(hist.current, wc) and np.array_equal(hist.previous, wp)
    else:
        assert abs(got.iterations - want.iterations) <= 1
        assert abs(got.r_initial - want.r_initial) <= 1e-14 * want.r_initial


def test_iterate_to_tolerance_elastic_mms_fast(port):
    """Elasticity with semi-implicit APT converges in the same count (+-1) as the oracle."""
    g = P.Grid.make3d(12, 9, 10, 2.0, 1.0, 1.0)
    E, _, _, f, bc = elastic_case(g, 0)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.2 * h, theta=1.0, form=1)
    z = np.zeros(3 * g.num_nodes)
    rc, want, _, _ = port.iterate_to_tolerance(1, g, bc, E, 0.3, f, z, z, 1, p, 1e-3, 3000)
    op = D.ElasticityOperator(g, E, 0.3, f, bc, mode=FAST)
    hist = D.StateHistory.of(z)
    got = D.iterate_to_tolerance(hist, op, 1, p, 1e-3, 3000)
    assert got.converged == want.converged
    assert abs(got.iterations - want.iterations) <= 1


@pytest.mark.parametrize("n_apt", [150, 230])
def test_elasticity3d_reckless_abort_step(n_apt):
    """check_finite cadence on the fused 3D path: a blowing-up APT solve aborts at
    the same check (a multiple of 100, or the last step) in FAST and REPLICA mode
    (kernels after the first non-finite step's check are skipped)."""
    g = P.Grid.make3d(40, 17, 12, 2.0, 1.0, 0.7)
    E = H.random_modulus(g, 2)
    f = H.sparse_loads(g, 3, 3)
    bc = H.elastic_bc(g, "x_hi")
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=40.0 * h, theta=1.0, n_apt=n_apt, n_pt=0, form=0)
    steps = []
    for mode in (REPLICA, FAST):
        op = D.ElasticityOperator(g, E, 0.3, f, bc, mode=mode)
        hist = D.StateHistory.of(H.random_field(3 * g.num_nodes, 9, -1e-3, 1e-3))
        with pytest.raises(D.NumericalAbort) as ei:
            D.hybrid_solve(hist, op, p)
        steps.append(ei.value.step)
    assert steps[0] == steps[1]
    assert steps[0] % 100 == 0 or steps[0] == n_apt


def _heat_ctx_solve(g, kappa, src, bc, T0, p, tblock):
    """hybrid_solve of a 2D heat problem with or without temporal blocking (PETTO_NO_TBLOCK)."""
    import os

    old = os.environ.get("PETTO_NO_TBLOCK")
    os.environ["PETTO_NO_TBLOCK"] = "0" if tblock else "1"
    try:
        op = D.HeatOperator(g, kappa, src, bc, mode=FAST)
    finally:
        if old is None:
            del os.environ["PETTO_NO_TBLOCK"]
        else:
            os.environ["PETTO_NO_TBLOCK"] = old
    hist = D.StateHistory(T0.copy(), T0.copy())
    step = None
    try:
        D.hybrid_solve(hist, op, p)
    except D.NumericalAbort as e:
        step = e.step
    return hist, step


@pytest.mark.parametrize("form,n_apt,n_pt", [(1, 137, 63), (0, 95, 0), (0, 0, 110)])
def test_heat2d_temporal_blocking_matches_per_step_solve(port, form, n_apt, n_pt):
    """The temporally blocked 2D heat solve (10 steps per grid barrier, shared-memory
    tiles with halo) against the per-step solve and the oracle: many tiles, ragged
    edges, a dense source, pinned faces, both APT forms, pure PT, and rounds that
    straddle the APT -> PT switch or end short of 10 steps."""
    g = P.Grid.make2d(203, 151, 2.0, 1.5)
    bc = P.BoundarySpec.all_faces(2, P.NEUMANN_ZERO)
    bc.face[0] = P.FaceCondition(P.DIRICHLET, 0.25, 0)
    bc.face[3] = P.FaceCondition(P.DIRICHLET, -0.5, 0)
    r = H.rng(5)
    kappa = np.maximum(1e-3, r.random(g.num_nodes) ** 2)
    src = r.uniform(-1.0, 1.0, g.num_nodes)
    T0 = r.uniform(-0.1, 0.1, g.num_nodes)
    e, v = P.make_constraints(g, bc, 1)
    T0[e] = v
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=n_apt, n_pt=n_pt, form=form)
    a, _ = _heat_ctx_solve(g, kappa, src, bc, T0, p, True)
    b, _ = _heat_ctx_solve(g, kappa, src, bc, T0, p, False)
    assert rel_err(a.current, b.current) < 1e-13 and rel_err(a.previous, b.previous) < 1e-13
    rc, wc, wp, _ = port.hybrid_solve(0, g, bc, kappa, 0.3, src, T0, T0, p)
    assert rc == 0 and rel_err(a.current, wc) < 1e-10 and rel_err(a.previous, wp) < 1e-10


def test_heat2d_temporal_blocking_abort_state():
    """An exploding 2D heat solve aborts at the same check_finite step with the same
    buffers (the state of that step) in the blocked and the per-step solve."""
    g = P.Grid.make2d(90, 70, 1.0, 1.0)
    bc = P.BoundarySpec.all_faces(2, P.DIRICHLET)
    T0 = H.rng(6).uniform(-1e-3, 1e-3, g.num_nodes)
    p = P.PTParams(dt_pt=5e-4, dt_apt=0.5 / 15, theta=1.0, n_apt=0, n_pt=5000)
    a, sa = _heat_ctx_solve(g, np.ones(g.num_nodes), np.ones(g.num_nodes), bc, T0, p, True)
    b, sb = _heat_ctx_solve(g, np.ones(g.num_nodes), np.ones(g.num_nodes), bc, T0, p, False)
    assert sa is not None and sa == sb and sa % 100 == 0
    same = (a.current == b.current) | (np.isnan(a.current) & np.isnan(b.current))
    assert same.all()


def _elastic2d_ctx_solve(g, E, f, bc, u0, p, tblock):
    """hybrid_solve of a 2D elasticity problem with or without temporal blocking."""
    import os

    old = os.environ.get("PETTO_NO_TBLOCK")
    os.environ["PETTO_NO_TBLOCK"] = "0" if tblock else "1"
    try:
        op = D.ElasticityOperator(g, E, 0.3, f, bc, mode=FAST)
    finally:
        if old is None:
            del os.environ["PETTO_NO_TBLOCK"]
        else:
            os.environ["PETTO_NO_TBLOCK"] = old
    hist = D.StateHistory(u0.copy(), u0.copy())
    step = None
    try:
        D.hybrid_solve(hist, op, p)
    except D.NumericalAbort as e:
        step = e.step
    return hist, step


@pytest.mark.parametrize("form,n_apt,n_pt", [(1, 137, 63), (0, 95, 0), (0, 0, 110), (1, 3, 2)])
def test_elastic2d_temporal_blocking_matches_per_step_solve(port, form, n_apt, n_pt):
    """The temporally blocked 2D elasticity solve (4 steps per grid barrier, 56 x 8
    tiles with a 4-node halo) against the per-step solve and the oracle: many tiles,
    ragged edges, a random modulus, point loads, a clamped face plus single-component
    pins, both APT forms, pure PT, rounds straddling the APT -> PT switch."""
    g = P.Grid.make2d(203, 77, 2.0, 0.8)
    E = H.random_modulus(g, 8)
    f = H.sparse_loads(g, 2, 9, count=40)
    bc = H.elastic_bc(g, "x_lo", pins=[(g.node(202, 0), 1, 0.0), (g.node(100, 40), 0, 0.01)])
    e, v = P.make_constraints(g, bc, 2)
    u0 = H.random_field(2 * g.num_nodes, 10, -1e-3, 1e-3)
    u0[e] = v
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=n_apt, n_pt=n_pt, form=form)
    a, _ = _elastic2d_ctx_solve(g, E, f, bc, u0, p, True)
    b, _ = _elastic2d_ctx_solve(g, E, f, bc, u0, p, False)
    assert rel_err(a.current, b.current) < 1e-13 and rel_err(a.previous, b.previous) < 1e-13
    assert np.array_equal(a.current[e], v)
    rc, wc, wp, _ = port.hybrid_solve(1, g, bc, E, 0.3, f, u0, u0, p)
    assert rc == 0 and rel_err(a.current, wc) < 1e-10 and rel_err(a.previous, wp) < 1e-10


def test_elastic2d_temporal_blocking_abort_state():
    """An exploding 2D elasticity solve aborts at the same check_finite step with the
    same buffers in the blocked and the per-step solve."""
    g = P.Grid.make2d(120, 50, 2.0, 1.0)
    E = H.random_modulus(g, 3)
    bc = H.elastic_bc(g, "x_lo")
    u0 = H.random_field(2 * g.num_nodes, 4, -1e-3, 1e-3)
    e, v = P.make_constraints(g, bc, 2)
    u0[e] = v
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=40.0 * h, theta=1.0, n_apt=2000, n_pt=0, form=0)
    a, sa = _elastic2d_ctx_solve(g, E, np.zeros(2 * g.num_nodes), bc, u0, p, True)
    b, sb = _elastic2d_ctx_solve(g, E, np.zeros(2 * g.num_nodes), bc, u0, p, False)
    assert sa is not None and sa == sb and sa % 100 == 0
    same = (a.current == b.current) | (np.isnan(a.current) & np.isnan(b.current))
    assert same.all()


@pytest.mark.parametrize("nx,ny", [(56, 24), (57, 25), (112, 48), (3, 150), (300, 3), (5, 3), (400, 200), (113, 430)])
def test_elastic2d_temporal_blocking_tile_edges(port, nx, ny):
    """Grids at, just past and far below the tile sizes (56 x 8 for grids that fit
    148 of them, else 56 x 24: the last two grids), single rows / columns of tiles,
    three-node-wide grids: blocked = per-step = oracle."""
    g = P.Grid.make2d(nx, ny, 1.0 + nx / 100.0, 1.0)
    E = H.random_modulus(g, nx + ny)
    f = H.sparse_loads(g, 2, 3, count=3)
    bc = H.elastic_bc(g, "x_lo" if nx > 3 else "y_lo")
    e, v = P.make_constraints(g, bc, 2)
    u0 = H.random_field(2 * g.num_nodes, 12, -1e-3, 1e-3)
    u0[e] = v
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=37, n_pt=9, form=1)
    a, _ = _elastic2d_ctx_solve(g, E, f, bc, u0, p, True)
    b, _ = _elastic2d_ctx_solve(g, E, f, bc, u0, p, False)
    assert rel_err(a.current, b.current) < 1e-13 and rel_err(a.previous, b.previous) < 1e-13
    rc, wc, wp, _ = port.hybrid_solve(1, g, bc, E, 0.3, f, u0, u0, p)
    assert rc == 0 and rel_err(a.current, wc) < 1e-10 and rel_err(a.previous, wp) < 1e-10


@pytest.mark.parametrize("mode", [FAST, REPLICA])
@pytest.mark.parametrize("gi", [1, 4])
def test_boundary_uploads_independent_of_order(port, gi, mode):
    """set_constraints / set_source in either order, and a second set_constraints
    with a different constraint set after the loads, give the same operator: the
    context rebuilds its pinned values and loads from its own copies of both."""
    g = ELASTIC_GRIDS[gi]
    d = g.dim
    E = H.random_modulus(g, 3)
    u = H.random_field(d * g.num_nodes, 21)
    f = H.sparse_loads(g, d, 5, count=40)
    bc_a = H.elastic_bc(g, "x_lo")
    bc_b = H.elastic_bc(g, "x_hi", pins=[(g.node(0, 0), 1, 0.25)])
    ea, va = P.make_constraints(g, bc_a, d)
    eb, vb = P.make_constraints(g, bc_b, d)
    want = port.elasticity_residual(g, bc_b, E, 0.3, f, u)
    outs = []
    for order in ("cons_first", "loads_first", "replaced"):
        ctx = D.Context(g, 1, 0.3, mode)
        if order == "cons_first":
            ctx.set_constraints(eb, vb)
            ctx.set_source(f)
        elif order == "loads_first":
            ctx.set_source(f)
            ctx.set_constraints(eb, vb)
        else:  # an earlier constraint set, the loads, then the real constraint set
            ctx.set_constraints(ea, va)
            ctx.set_source(f)
            ctx.set_constraints(eb, vb)
        ctx.set_property(E)
        ctx.init_operator()
        ctx.set_state(u, u)
        outs.append(ctx.residual()[0])
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    if mode == REPLICA:
        assert np.array_equal(outs[0], want)
    else:
        assert rel_err(outs[0], want) < 1e-12


def _elastic3d_solve(g, E, f, bc, u0, up0, p, multi):
    """hybrid_solve of a 3D elasticity problem, FAST, one persistent launch per form
    segment (PETTO_MULTI=1) or one launch per step (PETTO_MULTI=0)."""
    import os

    old = os.environ.get("PETTO_MULTI")
    os.environ["PETTO_MULTI"] = "1" if multi else "0"
    try:
        op = D.ElasticityOperator(g, E, 0.3, f, bc, mode=FAST)
    finally:
        if old is None:
            del os.environ["PETTO_MULTI"]
        else:
            os.environ["PETTO_MULTI"] = old
    hist = D.StateHistory(u0.copy(), up0.copy())
    step = None
    try:
        D.hybrid_solve(hist, op, p)
    except D.NumericalAbort as e:
        step = e.step
    return hist, step


PERSISTENT_CASES = [
    # grid, form, n_apt, n_pt
    (P.Grid.make3d(70, 23, 19, 2.0, 1.0, 1.0), 1, 37, 24),    # several x tiles and strips, ragged
    (P.Grid.make3d(12, 9, 10, 2.0, 1.0, 1.0), 0, 50, 0),
    (P.Grid.make3d(40, 17, 130, 2.0, 1.0, 0.7), 0, 0, 33),   # several z chunks, pure PT
    (P.Grid.make3d(128, 64, 64, 1.0, 1.0, 1.0), 1, 100, 100),  # C4's grid
    (P.Grid.make3d(33, 1100, 6, 1.0, 0.5, 1.0), 1, 20, 7),    # 158 strips: several items per CTA and step
]


@pytest.mark.parametrize("case", range(len(PERSISTENT_CASES)))
def test_elastic3d_persistent_matches_per_step_solve(port, case):
    """The persistent 3D solve (all steps of a form segment in one cooperative
    launch, grid barriers between them) is bit-identical to one launch per step,
    and agrees with the oracle."""
    g, form, n_apt, n_pt = PERSISTENT_CASES[case]
    E, u, up, f, bc = elastic_case(g, 4)
    e, v = P.make_constraints(g, bc, 3)
    u[e] = v
    up[e] = v
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.05 * h, theta=1.0, n_apt=n_apt, n_pt=n_pt, form=form)
    a, sa = _elastic3d_solve(g, E, f, bc, u, up, p, True)
    b, sb = _elastic3d_solve(g, E, f, bc, u, up, p, False)
    assert sa is None and sb is None
    assert np.array_equal(a.current, b.current) and np.array_equal(a.previous, b.previous)
    if g.num_nodes <= 33 * 1100 * 6:
        rc, wc, wp, _ = port.hybrid_solve(1, g, bc, E, 0.3, f, u, up, p)
        assert rc == 0 and rel_err(a.current, wc) < 1e-10 and rel_err(a.previous, wp) < 1e-10


@pytest.mark.parametrize("n_apt", [150, 230])
def test_elastic3d_persistent_abort_state(n_apt):
    """An exploding 3D solve aborts at the same check_finite step with the same
    buffers in the persistent and the per-step solve (the steps after the check
    are skipped inside the launch)."""
    g = P.Grid.make3d(40, 17, 12, 2.0, 1.0, 0.7)
    E = H.random_modulus(g, 2)
    f = H.sparse_loads(g, 3, 3)
    bc = H.elastic_bc(g, "x_hi")
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=40.0 * h, theta=1.0, n_apt=n_apt, n_pt=0, form=0)
    u0 = H.random_field(3 * g.num_nodes, 9, -1e-3, 1e-3)
    a, sa = _elastic3d_solve(g, E, f, bc, u0, u0, p, True)
    b, sb = _elastic3d_solve(g, E, f, bc, u0, u0, p, False)
    assert sa is not None and sa == sb
    assert np.array_equal(a.current, b.current, equal_nan=True)
    assert np.array_equal(a.previous, b.previous, equal_nan=True)


@pytest.mark.parametrize("mode", [REPLICA, FAST])
@pytest.mark.parametrize("c", [0.9050125313283208, 0.982])
def test_iterate_to_tolerance_divergence_abort(port, mode, c):
    """A diverging tolerance loop (explicit PT beyond its stability limit) aborts at
    the iteration whose residual norm is first non-finite (state_solver.hpp:531-533),
    like the reference -- also when that iteration is a multiple of 100, the
    hybrid solve's check_finite cadence (c = 0.905: the reference aborts at 200)."""
    g = P.Grid.make2d(24, 24, 1.0, 1.0)
    bc = P.BoundarySpec.all_faces(2, P.DIRICHLET)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h * c, dt_apt=h / 2, theta=1.0, form=0)
    z = np.zeros(g.num_nodes)
    one = np.ones(g.num_nodes)
    rc, want, _, _ = port.iterate_to_tolerance(0, g, bc, one, 0.3, one, z, z, 0, p, 1e-30, 1000)
    assert rc != 0
    op = D.HeatOperator(g, one, one, bc, mode=mode)
    hist = D.StateHistory.of(z)
    with pytest.raises(D.NumericalAbort) as ei:
        D.iterate_to_tolerance(hist, op, 0, p, 1e-30, 1000)
    assert ei.value.step == want.iterations


def _elastic3d_tol(g, E, f, bc, u0, p, target, max_iters, multi):
    import os

    old = os.environ.get("PETTO_MULTI")
    os.environ["PETTO_MULTI"] = "1" if multi else "0"
    try:
        op = D.ElasticityOperator(g, E, 0.3, f, bc, mode=FAST)
    finally:
        if old is None:
            del os.environ["PETTO_MULTI"]
        else:
            os.environ["PETTO_MULTI"] = old
    hist = D.StateHistory(u0.copy(), u0.copy())
    st = D.iterate_to_tolerance(hist, op, 1, p, target, max_iters)
    return hist, st


@pytest.mark.parametrize("gi,form,rel_target,max_iters", [(0, 1, 0.05, 5000), (1, 0, 0.2, 3000), (0, 1, 1e-9, 150),
                                                          (2, 1, 0.05, 20000)])
def test_elastic3d_persistent_tolerance_matches_per_step(gi, form, rel_target, max_iters):
    """iterate_to_tolerance in persistent launches (the stop test on the device after
    a grid barrier) against one launch per iteration + k_iter_finish: the same
    iterations, residual norms and state, bit for bit -- converged, and stopped by
    max_iters (third case)."""
    g = [P.Grid.make3d(12, 9, 10, 2.0, 1.0, 1.0), P.Grid.make3d(70, 23, 19, 2.0, 1.0, 1.0),
         P.Grid.make3d(128, 64, 64, 1.0, 1.0, 1.0)][gi]
    E, _, _, f, bc = elastic_case(g, 0)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.2 * h, theta=1.0, form=form)
    z = np.zeros(3 * g.num_nodes)
    op = D.ElasticityOperator(g, E, 0.3, f, bc, mode=FAST)
    r0 = op.residual(z)
    target = rel_target * np.sqrt(np.sum(r0 ** 2)) / g.num_nodes
    a, sa = _elastic3d_tol(g, E, f, bc, z, p, target, max_iters, True)
    b, sb = _elastic3d_tol(g, E, f, bc, z, p, target, max_iters, False)
    assert (sa.iterations, sa.converged, sa.r_initial, sa.r_final) == (sb.iterations, sb.converged, sb.r_initial,
                                                                       sb.r_final)
    assert sa.converged == (rel_target > 1e-6)
    assert np.array_equal(a.current, b.current) and np.array_equal(a.previous, b.previous)

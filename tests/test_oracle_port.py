"""Pin the plain-C restatement (oracle/liboracle.so) to the reference itself
(oracle/_ref/libpetto_ref.so, built from /root/reference sources).

Bitwise equality is required everywhere: the restatement follows the reference's
operation order and both are compiled without FMA contraction.  The reference runs
with threads = 1 (parallel.hpp:9-15: serial mode is the bit-exact mode).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2509_06971_b200 import problem as P

from . import helpers as H


@pytest.fixture(autouse=True)
def serial(ref):
    ref.set_threads(1)
    yield


def test_unit_cell_stiffness_bitwise(port, ref):
    for dim, h in [(2, (0.1, 0.05, 1.0)), (3, (2 / 511, 1 / 255, 1 / 255)), (3, (1.0, 0.8, 0.6))]:
        for nu in (0.3, 0.25):
            a = port.unit_cell_stiffness(dim, h, nu)
            b = ref.unit_cell_stiffness(dim, h, nu)
            assert np.array_equal(a, b)


def test_spectral_bound_and_ch_dt(port, ref):
    for g in H.grids():
        assert port.spectral_bound(g, 0.3, 2.0) == ref.spectral_bound(g, 0.3, 2.0)
        assert port.ch_stable_dt(g, 1.0, 3e-5) == ref.ch_stable_dt(g, 1.0, 3e-5)


def test_make_constraints_matches(port, ref):
    g = P.Grid.make2d(9, 7, 1.0, 1.0)
    bc = P.BoundarySpec.all_faces(2, P.DIRICHLET, 1.5)
    bc.face[1] = P.FaceCondition(P.ROLLER, 0.25, 1)
    for comps in (1, 2):
        bc.pins = [(3, 0, -2.0), (g.node(0, 0), comps - 1, 7.0)]
        e1, v1 = port.make_constraints(g, bc, comps)
        e2, v2 = ref.make_constraints(g, bc, comps)
        e3, v3 = P.make_constraints(g, bc, comps)
        assert np.array_equal(e1, e2) and np.array_equal(v1, v2)
        assert np.array_equal(e3, e2) and np.array_equal(v3, v2)


@pytest.mark.parametrize("gi", range(4))
def test_elasticity_residual_bitwise(port, ref, gi):
    g = H.grids()[gi]
    d = g.dim
    E = H.random_modulus(g, seed=gi + 1)
    u = H.random_field(d * g.num_nodes, seed=7 + gi)
    f = H.sparse_loads(g, d, seed=3 + gi)
    bc = H.elastic_bc(g, "x_hi", pins=[(g.node(0, 0), 1, 0.0)])
    a = port.elasticity_residual(g, bc, E, 0.3, f, u)
    b = ref.elasticity_residual(g, bc, E, 0.3, f, u)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("gi", range(4))
def test_heat_residual_bitwise(port, ref, gi):
    g = H.grids()[gi]
    kappa = H.rng(gi).uniform(0.5, 2.0, g.num_nodes)
    src = H.rng(gi + 9).uniform(-1, 1, g.num_nodes)
    T = H.random_field(g.num_nodes, 11 + gi, -1, 1)
    bc = H.heat_bc(g)
    assert np.array_equal(port.heat_residual(g, bc, kappa, src, T), ref.heat_residual(g, bc, kappa, src, T))


def test_invalid_inputs_raise_invalid_argument(port, ref):
    g = P.Grid.make2d(5, 5, 1.0, 1.0)
    bc = H.elastic_bc(g, None)
    E = np.ones(g.num_nodes)
    E[7] = 0.0
    for o in (port, ref):
        with pytest.raises(O.OracleError) as ei:
            o.elasticity_residual(g, bc, E, 0.3, np.zeros(2 * g.num_nodes), np.zeros(2 * g.num_nodes))
        assert ei.value.code == 2
        with pytest.raises(O.OracleError) as ei:
            o.heat_residual(g, H.heat_bc(g), E, np.zeros(g.num_nodes), np.zeros(g.num_nodes))
        assert ei.value.code == 2


@pytest.mark.parametrize("physics,form", [(0, 0), (0, 1), (1, 1), (1, 0)])
def test_hybrid_solve_bitwise(port, ref, physics, form):
    for g in (P.Grid.make2d(20, 12, 1.0, 1.0), P.Grid.make3d(9, 7, 6, 1.0, 0.8, 0.6)):
        comps = g.dim if physics else 1
        prop = H.random_modulus(g, 5) if physics else H.rng(4).uniform(0.5, 2.0, g.num_nodes)
        src = H.sparse_loads(g, comps, 2) if physics else np.full(g.num_nodes, 0.3)
        bc = H.elastic_bc(g, "x_lo") if physics else H.heat_bc(g)
        cur = H.random_field(comps * g.num_nodes, 1, -0.01, 0.01)
        prev = H.random_field(comps * g.num_nodes, 2, -0.01, 0.01)
        h = g.min_spacing()
        p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=37, n_pt=23, form=form)
        ra = port.hybrid_solve(physics, g, bc, prop, 0.3, src, cur, prev, p)
        rb = ref.hybrid_solve(physics, g, bc, prop, 0.3, src, cur, prev, p)
        assert ra[0] == rb[0] == 0
        assert np.array_equal(ra[1], rb[1]) and np.array_equal(ra[2], rb[2])


def test_hybrid_reckless_step_aborts(port, ref):
    """tests/test_state_solver.cpp:330-340 fault injection."""
    g = P.Grid.make2d(16, 16, 1.0, 1.0)
    bc = P.BoundarySpec.all_faces(2, P.DIRICHLET)
    p = P.PTParams(dt_pt=1e6, dt_apt=0.5 / 15, theta=1.0, n_apt=0, n_pt=5000, form=0)
    z = np.zeros(g.num_nodes)
    for o in (port, ref):
        rc, cur, prev, step = o.hybrid_solve(0, g, bc, np.ones(g.num_nodes), 0.3, np.ones(g.num_nodes), z, z, p)
        assert rc == 1 and step == 100


def test_iterate_to_tolerance_counts(port, ref):
    g = P.Grid.make2d(24, 24, 1.0, 1.0)
    bc = P.BoundarySpec.all_faces(2, P.DIRICHLET)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 4, dt_apt=h / 2, theta=1.0, form=0)
    z = np.zeros(g.num_nodes)
    for mode in (0, 1):
        a = port.iterate_to_tolerance(0, g, bc, np.ones(g.num_nodes), 0.3, np.ones(g.num_nodes), z, z, mode, p,
                                      1e-6, 100000)
        b = ref.iterate_to_tolerance(0, g, bc, np.ones(g.num_nodes), 0.3, np.ones(g.num_nodes), z, z, mode, p,
                                     1e-6, 100000)
        assert a[0] == b[0] == 0
        assert a[1].iterations == b[1].iterations and a[1].r_final == b[1].r_final
        assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])


def _mats(kind, P_):
    props = [1.0, 0.37, 0.2][:P_] if kind == 0 else [1.0, 0.42, 0.1][:P_]
    return O.material_struct(kind, props, 0.3, 3.0, 1e-6)


@pytest.mark.parametrize("kind", [0, 1])
def test_design_subsystems_bitwise(port, ref, kind):
    for g in (P.Grid.make2d(8, 8, 1.0, 1.0), P.Grid.make3d(6, 6, 6, 1.0, 1.0, 1.0), P.Grid.make2d(21, 13, 4.0, 1.0)):
        np_ = 2 if g.dim == 3 else 3
        mat = _mats(kind, np_)
        phases = H.rng(42).uniform(0.2, 0.8, np_ * g.num_nodes)
        comps = g.dim if kind else 1
        state = H.random_field(comps * g.num_nodes, 8, -0.15, 0.15)
        region = np.arange(0, g.num_nodes, 3, dtype=np.int64)
        tgt = O.targets_struct([0.3, 0.5, 0.2][:np_], region, [0.1, 0.9, 0.0][:np_])
        assert np.array_equal(port.interpolate(g, mat, phases), ref.interpolate(g, mat, phases))
        sa = port.sensitivities(g, mat, tgt, phases, state)
        sb = ref.sensitivities(g, mat, tgt, phases, state)
        for x, y in zip(sa, sb):
            assert np.array_equal(x, y)
        w = P.Weights(0.1, 3.0, 2.0, 1.5, True, -1)
        ua = port.design_update(g, np_, w, phases, *sa)
        ub = ref.design_update(g, np_, w, phases, *sb)
        assert np.array_equal(ua, ub)
        ra = port.evaluate_objectives(g, mat, tgt, phases, state)
        rb = ref.evaluate_objectives(g, mat, tgt, phases, state)
        for f in ("compliance", "volume", "unity", "region"):
            assert getattr(ra, f) == getattr(rb, f)
        assert list(ra.volume_fractions) == list(rb.volume_fractions)
        assert port.separation(g, np_, ua) == ref.separation(g, np_, ub)


def test_ch_step_bitwise(port, ref):
    for g in (P.Grid.make2d(32, 32, 1.0, 1.0), P.Grid.make3d(10, 8, 6, 1.0, 1.0, 1.0)):
        phi = H.rng(64).uniform(0.45, 0.55, g.num_nodes)
        h = g.min_spacing()
        for _ in range(3):
            a, sa = port.ch_step(g, 1.0, 3e-5, 500 * h ** 4, phi)
            b, sb = ref.ch_step(g, 1.0, 3e-5, 500 * h ** 4, phi)
            assert np.array_equal(a, b) and sa == sb
            phi = a
        assert port.gl_energy(g, phi, 3e-5) == ref.gl_energy(g, phi, 3e-5)


def _small(name, **kw):
    cfg = P.config(name)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


RUN_CASES = [
    ("C2", dict(nx=16, ny=16, n_apt=10, n_pt=10, max_loops=5, report_every=1)),
    ("C1", dict(nx=40, ny=20, max_loops=6, report_every=2)),
    ("C3", dict(nx=48, ny=24, max_loops=4, report_every=1)),
    ("C4", dict(nx=16, ny=8, nz=8, n_apt=30, n_pt=30, max_loops=3, report_every=1)),
]


@pytest.mark.parametrize("name,kw", RUN_CASES)
def test_run_loop_bitwise(port, ref, name, kw):
    cfg = _small(name, **kw)
    prob = P.build_problem(cfg)
    sched = P.build_schedule(cfg, prob.grid, spectral_bound=ref.spectral_bound)
    a = port.run(prob, sched)
    b = ref.run(prob, sched)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert len(a[2]) == len(b[2]) > 0
    for x, y in zip(a[2], b[2]):
        for f in ("loop", "apt_steps", "pt_steps", "compliance", "volume", "unity", "region", "r_pde", "separation"):
            assert getattr(x, f) == getattr(y, f), f
        assert list(x.volume_fractions) == list(y.volume_fractions)
    for f in ("loops", "apt_steps", "pt_steps", "design_updates", "ch_steps", "clamp_mass_drift", "termination"):
        assert getattr(a[3], f) == getattr(b[3], f), f

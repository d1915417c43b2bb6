"""GPU parity of the design subsystems and the coupled loop (SURVEY.md 8a rows
a19-a26) through the C-ABI, against the oracle (pinned to the reference).

REPLICA must match bit for bit except where libm's sin enters (the Cahn-Hilliard
double-well derivative: CUDA's sin and glibc's may differ in the last ulp, so CH
and everything downstream of it is checked to 1e-13).  FAST mode is checked per
call to 1e-12 relative and per loop inside the early window.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2509_06971_b200 import device as D
from paper_2509_06971_b200 import problem as P

from . import helpers as H

pytestmark = pytest.mark.gpu
FAST, REPLICA = D.MODE_FAST, D.MODE_REPLICA

GRIDS = [P.Grid.make2d(8, 8, 1.0, 1.0), P.Grid.make3d(6, 6, 6, 1.0, 1.0, 1.0), P.Grid.make2d(21, 13, 4.0, 1.0),
         P.Grid.make3d(35, 12, 9, 2.0, 1.0, 0.8)]


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def design_case(g, kind, np_):
    props = [1.0, 0.37, 0.2][:np_] if kind == 0 else [1.0, 0.42, 0.1][:np_]
    phases = H.rng(42).uniform(0.2, 0.8, np_ * g.num_nodes)
    comps = g.dim if kind else 1
    state = H.random_field(comps * g.num_nodes, 8, -0.15, 0.15)
    region = np.arange(0, g.num_nodes, 3, dtype=np.int64)
    fr, rf = [0.3, 0.5, 0.2][:np_], [0.1, 0.9, 0.0][:np_]
    w = P.Weights(0.1, 3.0, 2.0, 1.5, True, -1)
    return props, phases, state, region, fr, rf, w


def make_ctx(g, kind, mode, props, phases, state, region, fr, rf, w):
    ctx = D.Context(g, kind, 0.3, mode)
    ctx.set_design(kind, props, 0.3, 3.0, 1e-6, fr, w, region, rf)
    ctx.set_phases(phases)
    ctx.set_state(state, state)
    return ctx


@pytest.mark.parametrize("gi", range(len(GRIDS)))
@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("mode", [REPLICA, FAST])
def test_interpolate_update_objectives(port, gi, kind, mode):
    g = GRIDS[gi]
    np_ = 2 if g.dim == 3 else 3
    props, phases, state, region, fr, rf, w = design_case(g, kind, np_)
    mat = O.material_struct(kind, props, 0.3, 3.0, 1e-6)
    tgt = O.targets_struct(fr, region, rf)
    ctx = make_ctx(g, kind, mode, props, phases, state, region, fr, rf, w)
    # interpolate_into
    assert np.array_equal(ctx.interpolate(), port.interpolate(g, mat, phases))
    # objectives of the pre-update design
    rep, sep = ctx.objectives()
    want = port.evaluate_objectives(g, mat, tgt, phases, state)
    wsep = port.separation(g, np_, phases)
    got = [rep.compliance, rep.volume, rep.unity, rep.region] + list(rep.volume_fractions)[:np_]
    exp = [want.compliance, want.volume, want.unity, want.region] + list(want.volume_fractions)[:np_]
    if mode == REPLICA:
        assert got == exp and sep == wsep
    else:
        assert rel(got, exp) < 1e-12 and sep == wsep
    # sensitivities + design_update_inplace
    gc, gv, gu, gr = port.sensitivities(g, mat, tgt, phases, state)
    upd = port.design_update(g, np_, w, phases, gc, gv, gu, gr)
    ctx.design_update()
    got = ctx.get_phases()
    if mode == REPLICA:
        assert np.array_equal(got, upd)
    else:
        assert np.abs(got - upd).max() < 1e-12


@pytest.mark.parametrize("gi", [0, 2, 3])
@pytest.mark.parametrize("mode", [REPLICA, FAST])
def test_ch_step(port, gi, mode):
    g = GRIDS[gi]
    np_ = 2
    phi = H.rng(64).uniform(0.45, 0.55, np_ * g.num_nodes)
    h = g.min_spacing()
    dt = 0.5 * port.ch_stable_dt(g, 1.0, 3e-5)
    ctx = D.Context(g, 0, 0.3, mode)
    ctx.set_design(0, [1.0, 1e-6], 0.3, 3.0, 1e-6, [0.5, 0.5], P.Weights())
    ctx.set_phases(phi)
    for _ in range(3):
        stats = ctx.ch_step(1.0, 3e-5, dt)
        want = []
        for q in range(np_):
            phi_q, st = port.ch_step(g, 1.0, 3e-5, dt, phi[q * g.num_nodes:(q + 1) * g.num_nodes])
            phi[q * g.num_nodes:(q + 1) * g.num_nodes] = phi_q
            want.append(st)
        got = ctx.get_phases()
        assert np.abs(got - phi).max() <= 1e-14
        for a, b in zip(stats, want):
            assert rel(a, b) < 1e-13
        phi = got.copy()  # continue from the device state (no drift accumulation)
    del h


def test_pure_phases_are_ch_fixed_points():
    """tests/test_phase_field.cpp:65-75 / acceptance crit 8: pure phases stay put."""
    g = P.Grid.make2d(16, 12, 1.0, 1.0)
    for mode in (REPLICA, FAST):
        ctx = D.Context(g, 0, 0.3, mode)
        ctx.set_design(0, [1.0, 1e-6], 0.3, 3.0, 1e-6, [0.5, 0.5], P.Weights())
        phi = np.concatenate([np.ones(g.num_nodes), np.zeros(g.num_nodes)])
        ctx.set_phases(phi)
        ctx.ch_step(1.0, 3e-5, 1e-6)
        assert np.array_equal(ctx.get_phases(), phi)


RUN_CASES = [
    ("C2", dict(nx=16, ny=16, n_apt=10, n_pt=10, max_loops=5, report_every=1)),
    ("C1", dict(nx=40, ny=20, max_loops=6, report_every=2)),
    ("C3", dict(nx=48, ny=24, max_loops=4, report_every=1)),
    ("C4", dict(nx=16, ny=8, nz=8, n_apt=30, n_pt=30, max_loops=3, report_every=1)),
    ("C4", dict(nx=40, ny=17, nz=12, n_apt=40, n_pt=40, max_loops=3, report_every=1)),
]

REC_FIELDS = ("compliance", "volume", "unity", "region", "r_pde", "separation")


@pytest.mark.parametrize("case", range(len(RUN_CASES)))
@pytest.mark.parametrize("mode", [REPLICA, FAST])
def test_run_loop(port, case, mode):
    name, kw = RUN_CASES[case]
    cfg = P.config(name)
    for k, v in kw.items():
        setattr(cfg, k, v)
    prob = P.build_problem(cfg)
    sched = P.build_schedule(cfg, prob.grid, spectral_bound=D.spectral_bound)
    wph, wst, wrecs, wres = port.run(prob, sched)
    ctx = D.Context.from_problem(prob, mode)
    res, recs = ctx.run(sched)
    assert (res.loops, res.apt_steps, res.pt_steps, res.design_updates, res.ch_steps, res.termination) == (
        wres.loops, wres.apt_steps, wres.pt_steps, wres.design_updates, wres.ch_steps, wres.termination)
    assert len(recs) == len(wrecs)
    tol = 1e-12 if mode == REPLICA else 1e-9
    for a, b in zip(recs, wrecs):
        assert a.loop == b.loop and a.apt_steps == b.apt_steps
        for f in REC_FIELDS:
            x, y = getattr(a, f), getattr(b, f)
            assert abs(x - y) <= tol * max(abs(y), 1e-30) + 1e-300, (f, x, y)
        assert rel(list(a.volume_fractions), list(b.volume_fractions)) < tol
    assert rel(ctx.get_phases(), wph) < (1e-12 if mode == REPLICA else 1e-8)
    assert rel(ctx.get_state()[0], wst) < (1e-12 if mode == REPLICA else 1e-8)
    assert abs(res.clamp_mass_drift - wres.clamp_mass_drift) <= 1e-12 + 1e-9 * abs(wres.clamp_mass_drift)


def test_run_reckless_step_aborts(port):
    """tests/test_optimizer.cpp:122-131: a reckless dt ends the run with AbortedNaN."""
    cfg = P.config("C2", nx=16, ny=16, n_apt=0, n_pt=200, max_loops=3, report_every=1)
    cfg.dt_pt = 1e6
    prob = P.build_problem(cfg)
    sched = P.build_schedule(cfg, prob.grid, spectral_bound=D.spectral_bound)
    wph, wst, wrecs, wres = port.run(prob, sched)
    for mode in (REPLICA, FAST):
        ctx = D.Context.from_problem(prob, mode)
        res, recs = ctx.run(sched)
        assert res.termination == wres.termination == 2
        assert res.abort_detail == wres.abort_detail
        assert res.loops == wres.loops

"""CPU: the C restatement (and the Python assembly mirror) against golden fixtures
generated from the reference itself (tests/golden/make_golden.py)."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2509_06971_b200 import problem as P

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def crit1_inputs(n):
    g = P.Grid.make2d(n, n, 1.0, 1.0)
    bc = P.BoundarySpec.all_faces(2, P.DIRICHLET)
    i, j, _ = g.ijk()
    src = np.array([np.sin(np.pi * (g.spacing[0] * float(a))) * np.sin(np.pi * (g.spacing[1] * float(b)))
                    for a, b in zip(i, j)])
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 4.0, dt_apt=h / 2.0, theta=1.0, form=0)
    return g, bc, src, p


@pytest.mark.parametrize("n", [32, 64, 128])
def test_crit1_iteration_counts_port(port, n):
    """tests/acceptance.cpp:50-97 known answers: PT 3582/14810/60201, APT 1781/3448/6236."""
    gold = GOLDEN["crit1"][str(n)]
    g, bc, src, p = crit1_inputs(n)
    assert digest(src) == gold["source_digest"]
    z, one = np.zeros(g.num_nodes), np.ones(g.num_nodes)
    for mode, name in ((0, "pt"), (1, "apt")):
        rc, st, cur, _ = port.iterate_to_tolerance(0, g, bc, one, 0.3, src, z, z, mode, p, gold["target"], 4000000)
        assert rc == 0 and st.converged
        assert st.iterations == gold[name]["iterations"]
        assert st.r_final == gold[name]["r_final"]
        assert digest(cur) == gold[name]["state_digest"]


def elastic_case(gi):
    grids = [P.Grid.make2d(17, 9, 2.0, 1.0), P.Grid.make3d(12, 9, 10, 2.0, 1.0, 1.0),
             P.Grid.make3d(37, 15, 11, 2.0, 1.0, 0.7)]
    g = grids[gi]
    d = g.dim
    E = np.maximum(1e-6, np.random.default_rng(gi + 1).random(g.num_nodes) ** 3)
    u = np.random.default_rng(7 + gi).uniform(-0.1, 0.1, d * g.num_nodes)
    f = np.zeros(d * g.num_nodes)
    f[np.random.default_rng(3).choice(d * g.num_nodes, 5, replace=False)] = 0.5
    bc = P.BoundarySpec.all_faces(d, P.TRACTION_FREE)
    bc.face[1] = P.FaceCondition(P.DIRICHLET, 0.0, 0)
    bc.pins = [(g.node(0, 0), 1, 0.0)]
    p = P.PTParams(dt_pt=g.min_spacing() ** 2 / 8, dt_apt=0.1 * g.min_spacing(), theta=1.0, n_apt=37, n_pt=23,
                   form=1)
    return g, E, u, f, bc, p


@pytest.mark.parametrize("gi", range(3))
def test_elastic_digests_port(port, gi):
    gold = GOLDEN["kernels"][f"elastic_{gi}"]
    g, E, u, f, bc, p = elastic_case(gi)
    r = port.elasticity_residual(g, bc, E, 0.3, f, u)
    assert digest(r) == gold["residual_digest"]
    rc, cur, prev, _ = port.hybrid_solve(1, g, bc, E, 0.3, f, u * 0.1, u * 0.05, p)
    assert digest(cur) == gold["hybrid_cur_digest"] and digest(prev) == gold["hybrid_prev_digest"]


@pytest.mark.parametrize("key", sorted(GOLDEN["runs"]))
def test_run_histories_port(port, key):
    gold = GOLDEN["runs"][key]
    cfg = P.config(gold["config"], **gold["overrides"])
    prob = P.build_problem(cfg)
    sched = P.build_schedule(cfg, prob.grid, spectral_bound=port.spectral_bound)
    ph, st, recs, res = port.run(prob, sched)
    assert res.loops == gold["loops"] and res.termination == gold["termination"]
    assert res.clamp_mass_drift == gold["clamp_mass_drift"]
    assert len(recs) == len(gold["records"])
    for a, b in zip(recs, gold["records"]):
        for f in ("loop", "compliance", "volume", "unity", "region", "r_pde", "separation"):
            assert getattr(a, f) == b[f], f
        assert list(a.volume_fractions)[:prob.nphases] == b["volume_fractions"]
    assert digest(ph) == gold["phases_digest"] and digest(st) == gold["state_digest"]

"""CPU: the Python problem-assembly mirror (config -> Problem / LoopSchedule) against
the reference's parse_config + build_problem + build_schedule (golden JSON, and
live when oracle/_ref is present)."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2509_06971_b200 import device as D
from paper_2509_06971_b200 import problem as P

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))["assembly"]


def check(name, d):
    cfg = P.parse_config(d["text"])
    prob = P.build_problem(cfg)
    g = prob.grid
    sched = P.build_schedule(cfg, g, spectral_bound=D.spectral_bound)
    assert [g.dim] + g.n == [d["dim"]] + d["n"]
    assert g.spacing == d["spacing"]
    assert prob.physics == d["physics"]
    assert prob.properties == d["properties"] and prob.fractions == d["fractions"]
    assert (prob.poisson_ratio, prob.penalty, prob.void_floor) == (d["poisson_ratio"], d["penalty"], d["void_floor"])
    w = d["weights"]
    assert (prob.weights.alpha_compliance, prob.weights.alpha_volume, prob.weights.alpha_unity,
            prob.weights.alpha_region) == (w["alpha_compliance"], w["alpha_volume"], w["alpha_unity"],
                                           w["alpha_region"])
    assert int(prob.weights.normalize_compliance) == w["normalize_compliance"]
    assert prob.weights.compliance_sign == w["compliance_sign"]
    assert [[f.kind, f.value, f.component] for f in prob.bc.face] == d["faces"]
    assert [list(p) for p in prob.bc.pins] == [[a, b, c] for a, b, c in d["pins"]]
    s = d["schedule"]
    assert (sched.pt.dt_pt, sched.pt.dt_apt, sched.pt.theta, sched.pt.n_apt, sched.pt.n_pt, sched.pt.form) == (
        s["dt_pt"], s["dt_apt"], s["theta"], s["n_apt"], s["n_pt"], s["form"])
    assert (sched.ch_mobility, sched.ch_gamma, sched.dt_ch) == (s["ch_mobility"], s["ch_gamma"], s["dt_ch"])
    assert (sched.max_loops, sched.convergence_tol, sched.convergence_window, sched.report_every) == (
        s["max_loops"], s["convergence_tol"], s["convergence_window"], s["report_every"])
    if prob.physics == 1:
        nz = np.nonzero(prob.source)[0]
        assert [[int(e), float(prob.source[e])] for e in nz] == [[a, b] for a, b in d["source_nonzero"]]
    else:
        assert np.all(prob.source == d["source_value"])
    rn = prob.region_nodes if prob.has_region else np.zeros(0, np.int64)
    assert len(rn) == d["region_nodes_count"]
    assert hashlib.sha256(np.asarray(rn, np.int64).tobytes()).hexdigest() == d["region_nodes_digest"]
    changed = np.nonzero(prob.initial_state != d["initial_state"])[0]
    assert [[int(e), float(prob.initial_state[e])] for e in changed] == [[a, b] for a, b in
                                                                          d["initial_state_constrained"]]


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_assembly_matches_golden(name):
    check(name, GOLDEN[name])


def test_assembly_matches_reference_live(ref):
    from oracle import oracle as O

    text = P.CONFIGS["C1"].replace("nx = 160", "nx = 33")
    check("live", dict(O.ref_config_json(text), text=text, region_nodes_count=0,
                       region_nodes_digest=hashlib.sha256(b"").hexdigest()))


def test_c5_schedule_values():
    """dt_pt = 2.5531e-6 (h^2/6), dt_apt = 1.95695e-3 (h/2) at 512x256x256."""
    cfg = P.config("C5")
    g = P.make_grid(cfg)
    s = P.build_schedule(cfg, g, spectral_bound=D.spectral_bound)
    assert abs(s.pt.dt_pt - 2.5531e-6) < 1e-9 and abs(s.pt.dt_apt - 1.95695e-3) < 1e-8


def test_unknown_key_is_config_error():
    with pytest.raises(P.ConfigError):
        P.parse_config("preset = heat2d\nbogus = 1\n")

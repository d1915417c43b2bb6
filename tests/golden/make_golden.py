"""Generate the golden fixtures in tests/golden/ from the reference itself.

Run in a container where /root/reference is mounted (oracle/_ref is built from
it by `make -C oracle`):

    python tests/golden/make_golden.py

Every number here comes from the UNMODIFIED reference (oracle/_ref/libpetto_ref.so)
at threads = 1 (its bit-exact mode, parallel.hpp:9-15).  The fixtures pin the
C restatement (oracle/liboracle.so) and the device path on boxes where the
reference is absent.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2509_06971_b200 import problem as P  # noqa: E402


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def rng(seed):
    return np.random.default_rng(seed)


def assembly(ref):
    """ref_config_json for the presets and the BASELINE configs (small fields summarised)."""
    out = {}
    texts = {f"preset_{n}": f"preset = {n}\n" for n in ("heat2d", "mbb2d", "cantilever3d", "drone3d")}
    texts.update({k: v for k, v in P.CONFIGS.items() if k != "C5"})
    for name, text in texts.items():
        d = O.ref_config_json(text)
        rn = d.pop("region_nodes")
        d["region_nodes_count"] = len(rn)
        d["region_nodes_digest"] = hashlib.sha256(np.asarray(rn, np.int64).tobytes()).hexdigest()
        d["text"] = text
        out[name] = d
    return out


def crit1(ref):
    """tests/acceptance.cpp:50-97: PT/APT iteration counts to 1e-8 r0 (threads = 1)."""
    res = {}
    for n in (32, 64, 128):
        g = P.Grid.make2d(n, n, 1.0, 1.0)
        bc = P.BoundarySpec.all_faces(2, P.DIRICHLET)
        i, j, _ = g.ijk()
        # std::sin(pi * g.coord(a, i)) with coord = spacing * i, as acceptance.cpp:60-63
        src = np.array([np.sin(np.pi * (g.spacing[0] * float(ii))) * np.sin(np.pi * (g.spacing[1] * float(jj)))
                        for ii, jj in zip(i, j)])
        h = g.min_spacing()
        p = P.PTParams(dt_pt=h * h / 4.0, dt_apt=h / 2.0, theta=1.0, form=0)
        z = np.zeros(g.num_nodes)
        one = np.ones(g.num_nodes)
        r0 = ref.heat_residual(g, bc, one, src, z)
        target = 1e-8 * ref.residual_norm(r0, g.num_nodes, 1)
        row = {"target": target, "source_digest": digest(src)}
        for mode, name in ((0, "pt"), (1, "apt")):
            rc, st, cur, _ = ref.iterate_to_tolerance(0, g, bc, one, 0.3, src, z, z, mode, p, target, 4000000)
            row[name] = {"iterations": st.iterations, "r_initial": st.r_initial, "r_final": st.r_final,
                         "converged": st.converged, "state_digest": digest(cur)}
        res[str(n)] = row
        print("crit1", n, row["pt"]["iterations"], row["apt"]["iterations"], flush=True)
    return res


def kernels(ref):
    """Digests of residuals / hybrid_solve on seeded inputs (bit-exact pins)."""
    out = {}
    cases = [P.Grid.make2d(17, 9, 2.0, 1.0), P.Grid.make3d(12, 9, 10, 2.0, 1.0, 1.0),
             P.Grid.make3d(37, 15, 11, 2.0, 1.0, 0.7)]
    for gi, g in enumerate(cases):
        d = g.dim
        E = np.maximum(1e-6, rng(gi + 1).random(g.num_nodes) ** 3)
        u = rng(7 + gi).uniform(-0.1, 0.1, d * g.num_nodes)
        f = np.zeros(d * g.num_nodes)
        f[rng(3).choice(d * g.num_nodes, 5, replace=False)] = 0.5
        bc = P.BoundarySpec.all_faces(d, P.TRACTION_FREE)
        bc.face[1] = P.FaceCondition(P.DIRICHLET, 0.0, 0)
        bc.pins = [(g.node(0, 0), 1, 0.0)]
        r = ref.elasticity_residual(g, bc, E, 0.3, f, u)
        p = P.PTParams(dt_pt=g.min_spacing() ** 2 / 8, dt_apt=0.1 * g.min_spacing(), theta=1.0, n_apt=37, n_pt=23,
                       form=1)
        rc, cur, prev, _ = ref.hybrid_solve(1, g, bc, E, 0.3, f, u * 0.1, u * 0.05, p)
        out[f"elastic_{gi}"] = {"grid": [g.dim, g.n, g.length], "residual_digest": digest(r),
                                "residual_norm": ref.residual_norm(r, g.num_nodes, d),
                                "hybrid_cur_digest": digest(cur), "hybrid_prev_digest": digest(prev),
                                "hybrid_cur_absmax": float(np.abs(cur).max())}
    return out


RUN_CASES = [
    ("C2", dict(nx=16, ny=16, n_apt=10, n_pt=10, max_loops=5, report_every=1)),
    ("C1", dict(nx=40, ny=20, max_loops=6, report_every=2)),
    ("C3", dict(nx=48, ny=24, max_loops=4, report_every=1)),
    ("C4", dict(nx=16, ny=8, nz=8, n_apt=30, n_pt=30, max_loops=3, report_every=1)),
]


def runs(ref):
    out = {}
    for name, kw in RUN_CASES:
        cfg = P.config(name, **kw)
        prob = P.build_problem(cfg)
        sched = P.build_schedule(cfg, prob.grid, spectral_bound=ref.spectral_bound)
        ph, st, recs, res = ref.run(prob, sched)
        key = name + "_" + "_".join(f"{k}{v}" for k, v in kw.items())
        out[key] = {
            "config": name, "overrides": kw,
            "records": [{"loop": r.loop, "compliance": r.compliance, "volume": r.volume, "unity": r.unity,
                         "region": r.region, "r_pde": r.r_pde, "separation": r.separation,
                         "volume_fractions": list(r.volume_fractions)[:prob.nphases]} for r in recs],
            "loops": res.loops, "termination": res.termination, "clamp_mass_drift": res.clamp_mass_drift,
            "phases_digest": digest(ph), "state_digest": digest(st),
        }
    return out


def main():
    ref = O.load("reference")
    ref.set_threads(1)
    golden = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref (threads=1)",
              "assembly": assembly(ref), "kernels": kernels(ref), "runs": runs(ref), "crit1": crit1(ref)}
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(golden, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()

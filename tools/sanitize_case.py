"""Small invocations of the hot kernels for compute-sanitizer (tests/test_gpu_sanitize.py).

    compute-sanitizer --tool racecheck python tools/sanitize_case.py elastic3d

Cases: elastic3d (k_elastic3d_fast: TMA ring, mbarriers, TMEM hand-off,
setmaxnreg; both layouts, APT + PT + residual), elastic2d_tb (k_elastic2d_tb),
heat2d_tb (k_heat2d_tb), heat3d (k_small_solve<0>), group3 (3-slab local group:
peer-halo stores + stream flags, team reductions), design (the design-loop
kernels through run()).  No torch import: only this repo's kernels run."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_06971_b200 import device as D  # noqa: E402
from paper_2509_06971_b200 import problem as P  # noqa: E402
from paper_2509_06971_b200 import slab  # noqa: E402


def elastic_ctx(g, k_range=None, x_outermost=False):
    rng = np.random.default_rng(1)
    E = np.maximum(1e-6, rng.random(g.num_nodes) ** 3)
    bc = P.BoundarySpec.all_faces(g.dim, P.TRACTION_FREE)
    bc.face[1] = P.FaceCondition(P.DIRICHLET, 0.0, 0)
    f = np.zeros(g.dim * g.num_nodes)
    f[g.num_nodes + 5] = -1.0
    e, v = P.make_constraints(g, bc, g.dim)
    ctx = D.Context(g, 1, 0.3, k_range=k_range, x_outermost=x_outermost)
    ctx.set_constraints(e, v)
    ctx.set_source(f)
    ctx.set_property(E)
    ctx.init_operator()
    u = rng.uniform(-0.01, 0.01, g.dim * g.num_nodes)
    ctx.set_state(u, u)
    return ctx


def params(g, n_apt=6, n_pt=3, form=1):
    h = g.min_spacing()
    return P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=n_apt, n_pt=n_pt, form=form)


def main(case):
    if case == "elastic3d":
        g = P.Grid.make3d(70, 16, 12, 2.0, 1.0, 0.7)
        for xo in (False, True):
            ctx = elastic_ctx(g, x_outermost=xo)
            ctx.hybrid_solve(params(g))
            ctx.residual()
            ctx.iterate_to_tolerance(1, params(g), 0.0, 4)
    elif case == "elastic2d_tb":
        g = P.Grid.make2d(120, 40, 2.0, 1.0)
        elastic_ctx(g).hybrid_solve(params(g, 9, 4))
    elif case in ("heat2d_tb", "heat3d"):
        g = P.Grid.make2d(150, 90, 1.0, 1.0) if case == "heat2d_tb" else P.Grid.make3d(30, 20, 12, 1.0, 1.0, 1.0)
        bc = P.BoundarySpec.all_faces(g.dim, P.NEUMANN_ZERO)
        bc.face[0] = P.FaceCondition(P.DIRICHLET, 0.0, 0)
        e, v = P.make_constraints(g, bc, 1)
        ctx = D.Context(g, 0, 0.3)
        ctx.set_constraints(e, v)
        ctx.set_source(np.full(g.num_nodes, 0.5))
        ctx.set_property(np.random.default_rng(2).uniform(0.5, 2.0, g.num_nodes))
        ctx.init_operator()
        ctx.set_state(np.zeros(g.num_nodes))
        ctx.hybrid_solve(params(g, 23, 11, 0))
    elif case == "group3":
        g = P.Grid.make3d(40, 16, 15, 2.0, 1.0, 0.7)
        ctxs = [elastic_ctx(g, k_range=slab.slab_range(r, 3, g.n[2])) for r in range(3)]
        D.group_link(ctxs)
        D.group_hybrid_solve(ctxs, params(g))
        D.group_residual(ctxs)
    elif case == "design":
        cfg = P.config("C4", nx=24, ny=10, nz=10, n_apt=4, n_pt=4, max_loops=2, report_every=1)
        prob = P.build_problem(cfg)
        sched = P.build_schedule(cfg, prob.grid, spectral_bound=D.spectral_bound)
        for mode in (D.MODE_FAST, D.MODE_REPLICA):
            D.Context.from_problem(prob, mode).run(sched)
    else:
        raise SystemExit(f"unknown case {case}")
    print("case", case, "done")


if __name__ == "__main__":
    main(sys.argv[1])

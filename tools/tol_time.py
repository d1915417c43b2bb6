"""iterate_to_tolerance at C4 (APT, 2000 iterations): one launch per iteration +
k_iter_finish (PETTO_MULTI=0) against persistent launches with the stop test on
the device (PETTO_MULTI=1).  python tools/tol_time.py  (on a B200)"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2509_06971_b200 import device as D, problem as P
cfg = P.config("C4"); prob = P.build_problem(cfg)
sched = P.build_schedule(cfg, prob.grid, spectral_bound=D.spectral_bound)
N = prob.grid.num_nodes
for multi in ("0", "1", "0", "1"):
    os.environ["PETTO_MULTI"] = multi
    ctx = D.Context(prob.grid, prob.physics, prob.poisson_ratio, D.MODE_FAST, x_outermost=True)
    ctx.set_constraints(prob.cons_entry, prob.cons_value); ctx.set_source(prob.source)
    ctx.set_property(np.ones(N)); ctx.init_operator()
    z = np.zeros(3 * N)
    ctx.set_state(z, z)
    ctx.iterate_to_tolerance(1, sched.pt, 1e-30, 50)  # warm-up
    ctx.set_state(z, z)
    t0 = time.perf_counter()
    st = ctx.iterate_to_tolerance(1, sched.pt, 1e-30, 2000)
    dt = time.perf_counter() - t0
    print("multi", multi, "iters", st.iterations, "r_final", st.r_final, "ms", round(dt * 1e3, 2), "us/iter", round(dt * 1e6 / st.iterations, 2), flush=True)

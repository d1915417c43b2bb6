"""Device run() loop timing: the whole outer loop of
optimizer.hpp:184-219 on the device at C4 / C5, split into the state solve and
the rest (interpolate, sensitivities + update, Cahn-Hilliard, finiteness), beside
the reference's own loop (oracle/_ref, all host cores) on the same problem.

    python tools/run_loop_time.py C4 [loops] [--x] [--ref-loops K]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_06971_b200 import device as D  # noqa: E402
from paper_2509_06971_b200 import problem as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("loops", type=int, nargs="?", default=10)
ap.add_argument("--x", action="store_true", help="x-outermost device layout")
ap.add_argument("--ref-loops", type=int, default=0)
a = ap.parse_args()

cfg = P.config(a.config, max_loops=a.loops, report_every=10 ** 6)
prob = P.build_problem(cfg)
sched = P.build_schedule(cfg, prob.grid, spectral_bound=D.spectral_bound)
out = {"config": a.config, "loops": a.loops, "layout": "x-outermost" if a.x else "reference",
       "steps_per_loop": sched.pt.n_apt + sched.pt.n_pt}
import torch  # noqa: E402  (device synchronisation for the phase timers only)

# warm-up (module load, first launches)
D.Context.from_problem(P.build_problem(P.config(a.config, nx=24, ny=12, nz=12, max_loops=1)), x_outermost=a.x)
ctx = D.Context.from_problem(prob, x_outermost=a.x)
torch.cuda.synchronize()
t0 = time.perf_counter()
res, recs = ctx.run(sched)
torch.cuda.synchronize()
t_run = time.perf_counter() - t0
# the same loop phase by phase (optimizer.hpp:186-205), each phase timed alone
ctx = D.Context.from_problem(prob, x_outermost=a.x)
ctx.interpolate(download=False)
ctx.init_operator()
phases = {"interpolate": 0.0, "hybrid_solve": 0.0, "design_update": 0.0, "ch_step": 0.0}
calls = {"interpolate": lambda: ctx.interpolate(download=False), "hybrid_solve": lambda: ctx.hybrid_solve(sched.pt),
         "design_update": ctx.design_update,
         "ch_step": lambda: ctx.ch_step(sched.ch_mobility, sched.ch_gamma, sched.dt_ch)}
for _ in range(a.loops):
    for k, f in calls.items():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        phases[k] += time.perf_counter() - t0
per_loop = {k: v / a.loops * 1e3 for k, v in phases.items()}
tot = sum(per_loop.values())
out.update({"run_s": t_run, "per_loop_ms": t_run / a.loops * 1e3, "phase_ms_per_loop": per_loop,
            "solve_share": per_loop["hybrid_solve"] / tot, "records": len(recs), "termination": res.termination})
if a.ref_loops:
    from oracle import oracle as O

    if O.has_reference():
        ref = O.load("reference")
        ref.set_threads(len(os.sched_getaffinity(0)))
        rc = P.config(a.config, max_loops=a.ref_loops, report_every=10 ** 6)
        rp = P.build_problem(rc)
        rs = P.build_schedule(rc, rp.grid, spectral_bound=ref.spectral_bound)
        t0 = time.perf_counter()
        ref.run(rp, rs)
        tr = time.perf_counter() - t0
        out.update({"reference_per_loop_ms": tr / a.ref_loops * 1e3, "reference_threads": len(os.sched_getaffinity(0)),
                    "speedup_per_loop": (tr / a.ref_loops) / (t_run / a.loops)})
print(json.dumps(out))

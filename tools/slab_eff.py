"""Compute-side strong-scaling estimate on one B200: the fused step of one rank's
slab of C5 (interior slab: ghost planes on both sides) for N = 1, 2, 4, 8 ranks,
against 1/N of the whole-grid step.  The peer halo overlaps the exchange with
the step, so this is the per-step bound of the N-GPU run.

    python tools/slab_eff.py [z|x ...]   slabs along z (reference layout) and / or
                                         along x (x_outermost device layout)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_06971_b200 import device as D  # noqa: E402
from paper_2509_06971_b200 import problem as P  # noqa: E402
from paper_2509_06971_b200 import slab as SL  # noqa: E402

cfg = P.config("C5")
prob = P.build_problem(cfg)
sched = P.build_schedule(cfg, prob.grid, spectral_bound=D.spectral_bound)
g = prob.grid
E = np.maximum(1e-6, np.random.default_rng(1).random(g.num_nodes) ** 3)
steps = int(os.environ.get("STEPS", "40"))
params = P.PTParams(sched.pt.dt_pt, sched.pt.dt_apt, sched.pt.theta, steps, 0, sched.pt.form)


def measure(layout):
    res = {}
    axis = 0 if layout == "x" else 2
    for n in [int(v) for v in os.environ.get("NS", "1,2,4,8").split(",")]:
        r = n // 2 if n > 1 else 0  # an interior rank
        kr = SL.slab_range(r, n, g.n[axis]) if n > 1 else None
        ctx = D.Context(g, prob.physics, prob.poisson_ratio, D.MODE_FAST, k_range=kr, x_outermost=layout == "x")
        ctx.set_constraints(prob.cons_entry, prob.cons_value)
        ctx.set_source(prob.source)
        ctx.set_property(E)
        ctx.init_operator()
        ctx.set_state(prob.initial_state, prob.initial_state)
        ctx.hybrid_solve(params)  # warm-up
        stream = torch.cuda.ExternalStream(ctx.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.hybrid_solve(params)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
        res[n] = ms
        print(f"{layout}-slabs N={n} slab {kr} step {ms * 1e3:.1f} us  efficiency vs 1/N of N=1: "
              f"{res[min(res)] * min(res) / n / ms:.3f}", flush=True)
        del ctx
    return {"step_us": {k: v * 1e3 for k, v in res.items()}, "efficiency": {k: res[min(res)] * min(res) / k / v for k, v in res.items()}}


print(json.dumps({layout: measure(layout) for layout in (sys.argv[1:] or ["z", "x"])}))

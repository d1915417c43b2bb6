"""Per-CTA start/end of one fused C5 launch (probe build -DE3_CTA_TIMING):
spread of CTA durations and the tail (last end - first end)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_06971_b200 import device as D  # noqa: E402
from paper_2509_06971_b200 import problem as P  # noqa: E402

prob = P.build_problem(P.config("C5"))
sched = P.build_schedule(P.config("C5"), prob.grid, spectral_bound=D.spectral_bound)
ctx = D.Context.from_problem(prob)
E = np.maximum(1e-6, np.random.default_rng(1).random(prob.grid.num_nodes) ** 3)
ctx.set_property(E)
ctx.init_operator()
params = P.PTParams(sched.pt.dt_pt, sched.pt.dt_apt, sched.pt.theta, 20, 0, sched.pt.form)
ctx.hybrid_solve(params)
buf = (C.c_uint64 * 4096)()
assert D.lib().petto_dev_probe_cta_times(ctx.h, buf, 4096) == 0
a = np.array(buf[: 3 * 148], dtype=np.float64).reshape(148, 3)
slots = np.array(buf[1024: 1024 + 3 * 600], dtype=np.float64).reshape(600, 3)
t0 = a[:, 0].min()
start, end, sm = a[:, 0] - t0, a[:, 1] - t0, a[:, 2]
dur = end - start
print("kernel span us %.1f  CTA dur mean %.1f min %.1f max %.1f  start spread %.2f  end spread %.1f" %
      (end.max() / 1e3, dur.mean() / 1e3, dur.min() / 1e3, dur.max() / 1e3, start.max() / 1e3,
       (end.max() - end.min()) / 1e3))
order = np.argsort(dur)
print("slowest CTAs (block, sm, dur us):", [(int(i), int(sm[i]), round(dur[i] / 1e3, 1)) for i in order[-6:]])
print("fastest CTAs:", [(int(i), int(sm[i]), round(dur[i] / 1e3, 1)) for i in order[:6]])
# by item geometry: block b -> strip b % 37, chunk b // 37
for name, key in (("strip", np.arange(148) % 37), ("chunk", np.arange(148) // 37)):
    groups = {}
    for b in range(148):
        groups.setdefault(int(key[b]), []).append(dur[b] / 1e3)
    print(name, {k: round(float(np.mean(v)), 1) for k, v in sorted(groups.items())})

if slots[1, 0] > 0:  # slot probe (E3_SLOT_TIMING): CTA 0, cell warp 1
    n = int((slots[:, 1] > 0).sum())
    sl = slots[:n]
    arrive, leave, own = sl[:, 0], sl[:, 1], sl[:, 2]
    span = np.diff(leave)  # slot q: leave(q-1) -> leave(q)
    work = arrive[1:] - leave[:-1]  # warp 1's own work in slot q
    wait = leave[1:] - arrive[1:]   # its wait at the barrier
    o = own[1:] > 0
    print("slots %d: owned slot %.0f ns (work %.0f, barrier wait %.0f); prologue slot %.0f ns (work %.0f, wait %.0f)" %
          (n, span[o].mean(), work[o].mean(), wait[o].mean(), span[~o].mean(), work[~o].mean(), wait[~o].mean()))
    # slot right after a prologue (first owned task of a tile)
    after = np.where((~o[:-1]) & o[1:])[0] + 1
    print("first owned slot after a prologue %.0f ns; next owned %.0f ns" % (span[after].mean(), span[after + 1].mean()))

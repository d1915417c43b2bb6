"""Output-writer throughput at the C5 size, one B200.

    python tools/bench_writers.py [--nx 512 --ny 256 --nz 256] [--sample 4000000]

Writes the fields.vtk of a C5-sized 3D elasticity result (2 phases, the modulus,
3 displacement components = 6 arrays of N values, engine.cpp:178-189) through
petto_dev_write_vtk, (a) to /dev/null (device formatting + copy pipeline, no
disk) and (b) to a file (including the host file write), and the reference's own
write_vtk_structured_points (oracle/_ref, or the C port) on a bounded sample of
the same values, single-threaded as the reference writes.  Prints one JSON line.
"""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (the reference writer: baseline only)
from paper_2509_06971_b200 import device as D  # noqa: E402
from paper_2509_06971_b200 import problem as P  # noqa: E402


def main():
    a = argparse.ArgumentParser()
    a.add_argument("--nx", type=int, default=512)
    a.add_argument("--ny", type=int, default=256)
    a.add_argument("--nz", type=int, default=256)
    a.add_argument("--sample", type=int, default=4_000_000, help="values written by the reference writer")
    a.add_argument("--file", default=None, help="target of the on-disk run (default: a temp file)")
    args = a.parse_args()
    g = P.Grid.make3d(args.nx, args.ny, args.nz, 2.0, 1.0, 1.0)
    N = g.num_nodes
    rng = np.random.default_rng(7)
    ctx = D.Context(g, 1, 0.3, D.MODE_FAST)
    E = np.maximum(1e-6, rng.random(N) ** 3)
    ctx.set_property(E)
    u = rng.uniform(-0.1, 0.1, 3 * N)
    ctx.set_state(u, u)
    ctx.set_design(1, [1.0, 1e-6], 0.3, 3.0, 1e-6, [0.3, 0.7], P.Weights(0.1, 3.0, 2.0, 1.5, True, -1))
    ph = rng.uniform(0.0, 1.0, 2 * N)
    ctx.set_phases(ph)
    arrays = [(D.FIELD_PHASE, 0, "phase_0"), (D.FIELD_PHASE, 1, "phase_1"), (D.FIELD_PROPERTY, 0, "modulus")] + [
        (D.FIELD_STATE, c, "displacement_" + "xyz"[c]) for c in range(3)]
    values = 6 * N
    ctx.write_vtk(arrays, "/dev/null")  # warm-up (buffers, clocks)
    t0 = time.perf_counter()
    ctx.write_vtk(arrays, "/dev/null")
    t_null = time.perf_counter() - t0
    path = args.file or os.path.join(tempfile.gettempdir(), "petto_bench_fields.vtk")
    t0 = time.perf_counter()
    ctx.write_vtk(arrays, path)
    t_file = time.perf_counter() - t0
    size = os.path.getsize(path)
    os.remove(path)

    ref = O.load("reference") if O.has_reference() else O.load("port")
    ns = min(args.sample, N)
    gs = P.Grid.make3d(ns // (args.ny * 4) if ns >= args.ny * 4 * 3 else 3, args.ny, 4, 2.0, 1.0, 1.0)
    ns = gs.num_nodes
    vals = u[:ns]
    with tempfile.TemporaryDirectory() as d:
        t0 = time.perf_counter()
        ref.write_vtk(gs, [("displacement_x", vals)], os.path.join(d, "ref.vtk"))
        t_ref = time.perf_counter() - t0
    line = {
        "metric": "VTK writer throughput (fields.vtk of a C5-sized result)",
        "unit": "M values/s",
        "values": values,
        "bytes": size,
        "device_to_devnull": {"value": values / t_null / 1e6, "seconds": t_null,
                              "GB_per_s_text": size / t_null / 1e9},
        "device_to_file": {"value": values / t_file / 1e6, "seconds": t_file, "path": path},
        "reference": {"value": ns / t_ref / 1e6, "seconds": t_ref, "sample_values": ns, "cores": 1,
                      "kind": ref.name},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()

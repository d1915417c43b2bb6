"""`petto run` on the B200: tools/petto.cpp + run_cli
(src/engine.cpp:95-130, 224-269) without CLI11.

    python -m paper_2509_06971_b200 run --preset cantilever3d --out runs/c3d
    python -m paper_2509_06971_b200 run --config my.cfg --nx 512 --loops 50 --quiet

The same options, config format, output files and exit codes as the reference:
0 success, 2 config error (bad flags included), 3 numerical abort, 4 I/O error.
The optimisation runs on the device (petto_dev_run), the field files come from
the device writers (petto_dev_write_*), history.csv and summary.txt are written
as the reference writes them.  The device path computes in FP64 only, so
`precision = f32` is refused as a config error.  `--mode replica` selects the
reference-order kernels (parity runs); the default is the fused fast path.
"""
from __future__ import annotations

import argparse
import os
import sys

from . import device as D
from . import problem as P


class _ArgError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # bad flags are config errors (exit 2), as in tools/petto.cpp
        raise _ArgError(message)


def _g17(v: float) -> str:
    """fmt() of field_io.cpp:15-19 (snprintf "%.17g"); glibc spells negative NaN '-nan'."""
    if v != v:
        return "-nan" if _signbit(v) else "nan"
    return "%.17g" % v


def _g6(v: float) -> str:
    """std::ostream << double (default precision 6, %g)."""
    if v != v:
        return "-nan" if _signbit(v) else "nan"
    return "%g" % v


def _signbit(v: float) -> bool:
    import math

    return math.copysign(1.0, v) < 0


def resolve_config(a) -> P.ProblemConfig:
    """resolve_config (src/engine.cpp:95-130)."""
    if a.config:
        try:
            with open(a.config) as f:
                text = f.read()
        except OSError:
            raise P.ConfigError(f"cannot read config file '{a.config}'") from None
        cfg = P.parse_config(text)
        if a.preset:
            raise P.ConfigError("--preset and --config are mutually exclusive")
    elif a.preset:
        cfg = P.make_preset(a.preset)
    else:
        raise P.ConfigError("either --preset or --config is required")
    if a.nx is not None and a.nx > 0:
        cfg.nx = a.nx
    if a.ny is not None and a.ny > 0:
        cfg.ny = a.ny
    if a.nz is not None and a.nz > 0:
        cfg.nz = a.nz
    if a.loops is not None and a.loops > 0:
        cfg.max_loops = a.loops
    if a.out:
        cfg.out_dir = a.out
    if a.precision:
        cfg.precision = a.precision
    if a.threads is not None and a.threads >= 0:
        cfg.threads = a.threads
    if a.report_every is not None and a.report_every > 0:
        cfg.report_every = a.report_every
    if a.compliance_sign:
        cfg.compliance_sign = a.compliance_sign
    if not cfg.out_dir:
        cfg.out_dir = os.environ.get("PETTO_OUT", "")
    if not cfg.out_dir:
        raise P.ConfigError("no output directory: pass --out <dir> or set PETTO_OUT")
    P.validate_config(cfg)
    if cfg.precision == "f32":
        raise P.ConfigError("config field 'precision': the B200 path computes in f64 only")
    return cfg


TERMINATION = {0: "converged", 1: "max_loops", 2: "aborted_nan"}


def write_outputs(cfg, prob, sched, ctx, res, records, nphases):
    """write_outputs (src/engine.cpp:145-217); field files from the device buffers."""
    out = cfg.out_dir
    try:
        os.makedirs(out, exist_ok=True)
    except OSError:
        raise D.IoError(f"cannot create output directory '{out}'") from None
    join = lambda name: os.path.join(out, name)  # noqa: E731
    wants = lambda f: f in cfg.formats  # noqa: E731
    # history.csv (field_io.cpp:128-145)
    try:
        with open(join("history.csv"), "w") as f:
            f.write("loop,apt_steps,pt_steps,compliance,J_v,J_1,J_b,r_pde,separation")
            f.write("".join(f",volfrac_{i}" for i in range(nphases if records else 0)) + "\n")
            for r in records:
                f.write(f"{r.loop},{r.apt_steps},{r.pt_steps},{_g17(r.compliance)},{_g17(r.volume)},"
                        f"{_g17(r.unity)},{_g17(r.region)},{_g17(r.r_pde)},{_g17(r.separation)}")
                f.write("".join("," + _g17(r.volume_fractions[i]) for i in range(nphases)) + "\n")
    except OSError:
        raise D.IoError(f"cannot open '{join('history.csv')}' for writing") from None
    g = prob.grid
    ctx.interpolate(download=False)  # interpolate(result.phases, prob.material)
    thermal = prob.physics == 0
    prop_name = "conductivity" if thermal else "modulus"
    if g.dim == 2:
        for i in range(nphases):
            if wants("csv"):
                ctx.write_field_csv(D.FIELD_PHASE, i, join(f"phase_{i}.csv"))
            if wants("pgm"):
                ctx.write_pgm(D.FIELD_PHASE, i, join(f"phase_{i}.pgm"))
        if wants("csv"):
            ctx.write_field_csv(D.FIELD_PROPERTY, 0, join(prop_name + ".csv"))
        if wants("pgm"):
            ctx.write_pgm(D.FIELD_PROPERTY, 0, join(prop_name + ".pgm"))
        if thermal:
            ctx.write_field_csv(D.FIELD_STATE, 0, join("temperature.csv"))
        else:
            for c in range(g.dim):
                ctx.write_field_csv(D.FIELD_STATE, c, join(f"displacement_{'xyz'[c]}.csv"))
    else:
        arrays = [(D.FIELD_PHASE, i, f"phase_{i}") for i in range(nphases)] + [(D.FIELD_PROPERTY, 0, prop_name)]
        arrays += [(D.FIELD_STATE, c, f"displacement_{'xyz'[c]}") for c in range(prob.comps)]
        ctx.write_vtk(arrays, join("fields.vtk"))
    w = P.effective_weights(cfg, g)
    lines = [f"preset = {cfg.preset or '(custom)'}", f"termination = {TERMINATION.get(res.termination, 'unknown')}"]
    detail = bytes(res.abort_detail).split(b"\0", 1)[0].decode()
    if detail:
        lines.append(f"abort_detail = {detail}")
    lines += [f"loops = {res.loops}", f"apt_steps = {res.apt_steps}", f"pt_steps = {res.pt_steps}",
              f"design_updates = {res.design_updates}", f"ch_steps = {res.ch_steps}",
              f"clamp_mass_drift = {_g6(res.clamp_mass_drift)}", f"dt_pt = {_g6(sched.pt.dt_pt)}",
              f"dt_apt = {_g6(sched.pt.dt_apt)}", f"dt_ch = {_g6(sched.dt_ch)}",
              f"alpha_volume_effective = {_g6(w.alpha_volume)}", f"alpha_unity_effective = {_g6(w.alpha_unity)}",
              f"alpha_region_effective = {_g6(w.alpha_region)}"]
    if records:
        r = records[-1]
        lines += [f"final_compliance = {_g6(r.compliance)}", f"final_r_pde = {_g6(r.r_pde)}",
                  f"final_separation = {_g6(r.separation)}"]
        lines += [f"final_volfrac_{i} = {_g6(r.volume_fractions[i])}" for i in range(nphases)]
        lines.append(f"wall_seconds = {_g6(r.wall_seconds)}")
    try:
        with open(join("summary.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")
    except OSError:
        raise D.IoError("cannot write run summary") from None


def run(a) -> int:
    cfg = resolve_config(a)
    prob = P.build_problem(cfg)
    sched = P.build_schedule(cfg, prob.grid, spectral_bound=D.spectral_bound)
    ctx = D.Context.from_problem(prob, mode=D.MODE_REPLICA if a.mode == "replica" else D.MODE_FAST,
                                 device=a.device)

    def progress(r):
        if a.quiet:
            return
        fr = " ".join("%.3f" % r.volume_fractions[i] for i in range(prob.nphases))
        print("loop %6d  J=%.6e  r_pde=%.3e  sep=%.3f  volfrac=[%s]" % (r.loop, r.compliance, r.r_pde,
                                                                         r.separation, fr), flush=True)

    res, records = ctx.run(sched, progress)
    write_outputs(cfg, prob, sched, ctx, res, records, prob.nphases)
    if res.termination == 2:
        detail = bytes(res.abort_detail).split(b"\0", 1)[0].decode()
        print(f"aborted: {detail}", file=sys.stderr)
        return 3
    if not a.quiet:
        print(f"done: {TERMINATION.get(res.termination, 'unknown')} after {res.loops} loops")
    return 0


def main(argv=None) -> int:
    ap = _Parser(prog="python -m paper_2509_06971_b200",
                 description="pseudo-transient topology optimization on structured grids (B200)")
    sub = ap.add_subparsers(dest="cmd")
    r = sub.add_parser("run", help="run an optimization")
    r.add_argument("--preset", default="", help="preset name (heat2d, mbb2d, cantilever3d, drone3d)")
    r.add_argument("--config", default="", help="config file path")
    r.add_argument("--nx", type=int)
    r.add_argument("--ny", type=int)
    r.add_argument("--nz", type=int)
    r.add_argument("--loops", type=int, help="override the loop budget")
    r.add_argument("--out", default="", help="output directory (default: $PETTO_OUT)")
    r.add_argument("--precision", default="", help="f32 or f64 (the device path runs f64)")
    r.add_argument("--threads", type=int, help="accepted for compatibility (host threads are not used)")
    r.add_argument("--report-every", type=int)
    r.add_argument("--compliance-sign", default="")
    r.add_argument("--quiet", action="store_true")
    r.add_argument("--mode", choices=["fast", "replica"], default="fast")
    r.add_argument("--device", type=int, default=0)
    try:
        a = ap.parse_args(argv)
        if a.cmd != "run":
            raise _ArgError("a subcommand is required: run")
        if a.compliance_sign:
            if a.compliance_sign in ("+1", "1"):
                a.compliance_sign = 1
            elif a.compliance_sign == "-1":
                a.compliance_sign = -1
            else:
                print("config error: --compliance-sign must be +1 or -1", file=sys.stderr)
                return 2
        else:
            a.compliance_sign = 0
    except _ArgError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    try:
        return run(a)
    except P.ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except D.NumericalAbort as e:
        print(f"numerical abort: {e}", file=sys.stderr)
        return 3
    except D.IoError as e:
        print(f"i/o error: {e}", file=sys.stderr)
        return 4


if __name__ == "__main__":
    sys.exit(main())

"""`python -m paper_2509_06971_b200 run` (tools/petto.cpp,
src/engine.cpp:95-269).

CPU: config resolution and validation against the reference's parse_config /
validate_config (same ConfigError messages), flag errors and exit codes.
GPU: whole runs of small presets -- the reference's set of output files, the
history against the oracle's run() (replica bit-close, fast within the early
window), the field files against the oracle's final fields.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_2509_06971_b200 import cli
from paper_2509_06971_b200 import problem as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

BAD = [
    "nx = 2", "ny = 1", "nz = 2", "length_x = 0", "properties = 1, -1", "penalty = 0.5", "void_floor = 0",
    "poisson_ratio = 0.5", "target_fractions = 0.9, 0.3", "target_fractions = 0.5", "alpha_compliance = -1",
    "compliance_sign = 2", "n_apt = 0\nn_pt = 0", "theta = 0", "apt_form = implicit", "ch_gamma = 0",
    "dt_pt = -1", "max_loops = 0", "convergence_window = 1", "report_every = 0", "fixed_faces = z_lo",
    "load_count = 1\nload_0_box = 0,0,0,99,0,0\nload_0_direction = 0,-1,0\nload_0_magnitude = 1",
    "load_count = 1\nload_0_box = 0,0,0,1,0,0\nload_0_direction = 0,0,0\nload_0_magnitude = 1",
    "precision = f16", "threads = -2", "initial_phase = 1.5",
]


@pytest.mark.parametrize("extra", BAD)
def test_validate_config_messages_match_reference(extra):
    text = "preset = mbb2d\nnx = 40\nny = 16\n" + extra + "\n"
    if not O.has_reference():
        pytest.skip("oracle/_ref not built")
    want = O.ref_check_config(text)
    assert want is not None
    with pytest.raises(P.ConfigError) as e:
        P.validate_config(P.parse_config(text))
    assert str(e.value) == want


def test_valid_presets_pass_validation():
    for name in ("heat2d", "mbb2d", "cantilever3d", "drone3d"):
        P.validate_config(P.make_preset(name))


def _cli(*args, env=None):
    return subprocess.run([sys.executable, "-m", "paper_2509_06971_b200", *args], capture_output=True, text=True,
                          cwd=ROOT, env=env, timeout=600)


def test_cli_config_errors(tmp_path):
    env = dict(os.environ)
    env.pop("PETTO_OUT", None)
    r = _cli("run", "--preset", "mbb2d", env=env)
    assert r.returncode == 2 and "no output directory" in r.stderr
    cfg = tmp_path / "a.cfg"
    cfg.write_text("preset = heat2d\n")
    r = _cli("run", "--preset", "mbb2d", "--config", str(cfg), "--out", str(tmp_path))
    assert r.returncode == 2 and "mutually exclusive" in r.stderr
    r = _cli("run", "--out", str(tmp_path))
    assert r.returncode == 2 and "either --preset or --config" in r.stderr
    r = _cli("run", "--preset", "mbb2d", "--out", str(tmp_path), "--compliance-sign", "3")
    assert r.returncode == 2 and "--compliance-sign must be +1 or -1" in r.stderr
    r = _cli("run", "--preset", "mbb2d", "--out", str(tmp_path), "--bogus")
    assert r.returncode == 2
    r = _cli("run", "--preset", "mbb2d", "--out", str(tmp_path), "--nx", "2")
    assert r.returncode == 2 and "config field 'nx'" in r.stderr
    r = _cli("run", "--preset", "mbb2d", "--out", str(tmp_path), "--precision", "f32")
    assert r.returncode == 2 and "f64 only" in r.stderr
    cfg.write_text("preset = heat2d\nnot_a_key = 1\n")
    r = _cli("run", "--config", str(cfg), "--out", str(tmp_path))
    assert r.returncode == 2 and "unknown config key" in r.stderr


# ------------------------------------------------------------------- GPU runs

CASES = {
    "heat2d": "preset = heat2d\nnx = 33\nny = 29\nmax_loops = 3\nreport_every = 1\nn_apt = 30\nn_pt = 30\n",
    "mbb2d": "preset = mbb2d\nnx = 40\nny = 16\nproperties = 1, 0.55, 1e-6\ntarget_fractions = 0.2, 0.2, 0.6\n"
             "max_loops = 3\nreport_every = 1\nn_apt = 20\nn_pt = 20\nformats = csv, pgm\n",
    "cantilever3d": "preset = cantilever3d\nnx = 20\nny = 9\nnz = 7\nlength_x = 2\nlength_y = 1\nlength_z = 1\n"
                    "properties = 1, 1e-6\ntarget_fractions = 0.3, 0.7\nmax_loops = 3\nreport_every = 1\n"
                    "n_apt = 20\nn_pt = 20\n",
    "drone3d": "preset = drone3d\nnx = 24\nny = 12\nnz = 24\nmax_loops = 3\nreport_every = 1\nn_apt = 20\nn_pt = 20\n",
}
FILES = {
    "heat2d": {"history.csv", "summary.txt", "phase_0.csv", "phase_0.pgm", "phase_0.pgm.scale.txt", "phase_1.csv",
               "phase_1.pgm", "phase_1.pgm.scale.txt", "conductivity.csv", "conductivity.pgm",
               "conductivity.pgm.scale.txt", "temperature.csv"},
    "mbb2d": {"history.csv", "summary.txt"} | {f"phase_{i}.{e}" for i in range(3) for e in ("csv", "pgm", "pgm.scale.txt")}
             | {"modulus.csv", "modulus.pgm", "modulus.pgm.scale.txt", "displacement_x.csv", "displacement_y.csv"},
    "cantilever3d": {"history.csv", "summary.txt", "fields.vtk"},
    "drone3d": {"history.csv", "summary.txt", "fields.vtk"},
}


def _csv_values(path):
    with open(path) as f:
        lines = f.read().splitlines()
    return np.array([float(x) for ln in lines[1:] for x in ln.split(",")])


def _vtk_arrays(path):
    out, cur = {}, None
    with open(path) as f:
        for ln in f:
            if ln.startswith("SCALARS "):
                cur = ln.split()[1]
                out[cur] = []
            elif cur and not ln.startswith("LOOKUP_TABLE"):
                out[cur].append(float(ln))
    return {k: np.array(v) for k, v in out.items()}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("mode", ["replica", "fast"])
def test_cli_run_against_oracle(port, tmp_path, name, mode):
    cfgp = tmp_path / "run.cfg"
    cfgp.write_text(CASES[name])
    out = tmp_path / "out"
    r = _cli("run", "--config", str(cfgp), "--out", str(out), "--mode", mode)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "done: " in r.stdout
    assert set(os.listdir(out)) == FILES[name]
    cfg = P.parse_config(CASES[name])
    prob = P.build_problem(cfg)
    from paper_2509_06971_b200 import device as D

    sched = P.build_schedule(cfg, prob.grid, spectral_bound=D.spectral_bound)
    phases, state, recs, res = port.run(prob, sched)
    hist = np.loadtxt(out / "history.csv", delimiter=",", skiprows=1, ndmin=2)
    assert hist.shape[0] == len(recs)
    tol = 1e-11 if mode == "replica" else 1e-8
    for row, rec in zip(hist, recs):
        assert int(row[0]) == rec.loop
        assert abs(row[3] - rec.compliance) <= tol * abs(rec.compliance)
        for i in range(prob.nphases):
            assert abs(row[9 + i] - rec.volume_fractions[i]) <= tol
    with open(out / "summary.txt") as f:
        summ = dict(ln.split(" = ", 1) for ln in f.read().splitlines())
    assert summ["loops"] == str(res.loops) and summ["termination"] == cli.TERMINATION[res.termination]
    N = prob.grid.num_nodes
    ftol = 1e-9 if mode == "replica" else 1e-6
    if prob.grid.dim == 2:
        for i in range(prob.nphases):
            assert np.abs(_csv_values(out / f"phase_{i}.csv") - phases[i * N:(i + 1) * N]).max() <= ftol
    else:
        arr = _vtk_arrays(out / "fields.vtk")
        prop = "modulus" if prob.physics else "conductivity"
        comps = ["displacement_" + "xyz"[c] for c in range(prob.comps)]  # engine.cpp:183-185, heat too
        assert list(arr) == [f"phase_{i}" for i in range(prob.nphases)] + [prop] + comps
        for i in range(prob.nphases):
            assert np.abs(arr[f"phase_{i}"] - phases[i * N:(i + 1) * N]).max() <= ftol
        for c in range(prob.comps):
            u = state[c * N:(c + 1) * N]
            assert np.abs(arr[comps[c]] - u).max() <= ftol * max(1.0, np.abs(u).max())

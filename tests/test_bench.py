"""CPU: the measurement contract of bench.py -- algorithmic bytes per
node-update, one config dict for both arms, and the reference arm's JSON line
(oracle/_ref on the host cores, no product library loaded)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2509_06971_b200 import problem as P  # noqa: E402


@pytest.mark.parametrize("name,apt,pt", [("C5", 80, 56), ("C4", 80, 56), ("C1", 56, 40), ("C3", 56, 40),
                                         ("C2", 32, 24)])
def test_step_bytes_per_physics(name, apt, pt):
    """u_n, u_{n-1}, the property and u_{n+1}: 3D elasticity 80 B, 2D 56 B, heat 32 B."""
    prob = P.build_problem(P.config(name, nx=8, ny=8, nz=8) if name in ("C4", "C5") else P.config(name, nx=8, ny=8))
    assert bench.step_bytes(prob, 0) == bench.step_bytes(prob, 1) == apt
    assert bench.step_bytes(prob, 2) == pt


def test_reference_arm_line():
    """--impl reference: the same metric / unit / config dict as our arm, the
    reference's CPU path timed on the host, e2e = the line's own value."""
    from oracle import oracle as O

    if not O.has_reference():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == "GLUPS"
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"] and d["cpu_baseline"]["kind"] == "reference"

    class A:
        config, n_apt = "C1", 100

    cfg = P.config("C1")
    prob = P.build_problem(cfg)
    sched = P.build_schedule(cfg, prob.grid, spectral_bound=O.load("reference").spectral_bound)
    assert d["config"] == bench.config_dict(A, cfg, prob, sched, 1)
    assert "paper_2509_06971_b200/lib" not in r.stderr

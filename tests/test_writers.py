"""Output writers (field_io.cpp:15-126).

CPU part: the C restatement of the writers against the reference's own
write_field_csv / write_pgm / write_vtk_structured_points (byte for byte), and
the device "%.17g" formatter (csrc/g17.cuh) compiled for the host against glibc's
snprintf.  GPU part (test_gpu_writers.py): the device writers against the port.
"""
import os
import subprocess

import numpy as np
import pytest

from paper_2509_06971_b200 import problem as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def special_field(n, seed):
    """Values across the whole double range plus the cases %.17g treats specially."""
    r = np.random.default_rng(seed)
    v = r.uniform(-1.0, 1.0, n) * 10.0 ** r.integers(-30, 30, n)
    bits = r.integers(0, 2**63, n // 8, dtype=np.int64)
    v[: n // 8] = bits.view(np.float64)  # random bit patterns (subnormals, huge, NaN payloads)
    specials = [0.0, -0.0, np.inf, -np.inf, np.nan, -np.nan, 5e-324, 1e-4, 9.9999999999999995e-5, 1e16, 1e17,
                0.1, 1.0 / 3.0, 123.456, 1.7976931348623157e308, 2.2250738585072014e-308]
    v[n // 8: n // 8 + len(specials)] = specials
    return v


GRIDS = [P.Grid.make2d(37, 11, 2.0, 1.0), P.Grid.make3d(19, 7, 5, 2.0, 1.0, 0.7)]


def read(path):
    with open(path, "rb") as f:
        return f.read()


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_port_writers_match_reference(port, ref, tmp_path, gi):
    g = GRIDS[gi]
    v = special_field(g.num_nodes, 3 + gi)
    w = np.random.default_rng(9).uniform(0, 1, g.num_nodes)
    for impl in (port, ref):
        impl.write_field_csv(g, v, tmp_path / f"{impl.name}.csv")
        impl.write_vtk(g, [("phase_0", w), ("modulus", v)], tmp_path / f"{impl.name}.vtk")
    assert read(tmp_path / "port.csv") == read(tmp_path / "reference.csv")
    assert read(tmp_path / "port.vtk") == read(tmp_path / "reference.vtk")
    if g.dim == 2:
        for impl in (port, ref):
            impl.write_pgm(g, v, tmp_path / f"{impl.name}.pgm")
        assert read(tmp_path / "port.pgm") == read(tmp_path / "reference.pgm")
        assert read(tmp_path / "port.pgm.scale.txt") == read(tmp_path / "reference.pgm.scale.txt")


def test_port_writer_errors(port, tmp_path):
    g = GRIDS[1]
    from oracle.oracle import OracleError

    with pytest.raises(OracleError) as e:
        port.write_field_csv(g, np.zeros(g.num_nodes), tmp_path / "missing_dir" / "x.csv")
    assert e.value.code == 4 and "cannot open" in str(e.value)
    with pytest.raises(OracleError) as e:
        port.write_pgm(g, np.zeros(g.num_nodes), tmp_path / "x.pgm")
    assert "only 2D" in str(e.value)


def test_g17_formatter_matches_snprintf(tmp_path):
    """The device formatter's host build against glibc snprintf("%.17g") on ~10M values:
    special values, every power of two and of ten and their neighbours, exact decimal
    ties, random bit patterns and typical field magnitudes."""
    exe = tmp_path / "test_g17"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_2509_06971_b200", "csrc"), "-o",
                    str(exe), os.path.join(ROOT, "tests", "cpp", "test_g17.cpp")], check=True)
    r = subprocess.run([str(exe), "2000000", "4242"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "0 mismatches" in r.stdout

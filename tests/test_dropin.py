"""The C++ drop-in (include/petto_dev.hpp) used from the reference's own API.

CPU: compiles tests/cpp/test_dropin.cpp against the reference headers and sources
(only where /root/reference is mounted).  GPU: runs the prebuilt binary, which
compares petto::dev::{run, hybrid_solve, iterate_to_tolerance} with the
reference's petto::{run, hybrid_solve, iterate_to_tolerance} in one process."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "_build", "test_dropin")


def test_dropin_compiles_against_reference():
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference headers not mounted here")
    from paper_2509_06971_b200 import build

    build.build()
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_against_reference_on_gpu():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/test_dropin not built (needs /root/reference at build time)")
    res = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "ALL PASSED" in res.stdout

"""GPU: the output writers from device buffers against
the C restatement of the reference's writers (itself pinned byte for byte to the
reference in tests/test_writers.py): CSV, VTK and PGM files must be identical,
including NaN / inf / -0.0 / subnormal values, padded rows, multi-chunk fields,
and the reference's IoError."""
import numpy as np
import pytest

from paper_2509_06971_b200 import device as D
from paper_2509_06971_b200 import problem as P

from . import helpers as H
from .test_writers import special_field

pytestmark = pytest.mark.gpu
S, PH, PR = D.FIELD_STATE, D.FIELD_PHASE, D.FIELD_PROPERTY


def read(path):
    with open(path, "rb") as f:
        return f.read()


def test_format_values_matches_printf():
    ctx = D.Context(P.Grid.make2d(5, 5, 1.0, 1.0), 0, 0.3, D.MODE_FAST)
    v = special_field(300000, 11)
    got = ctx.format_values(v)
    # Python's %-formatting is correctly rounded like glibc's; only NaN differs (glibc: "-nan")
    want = "".join(("-nan\n" if (x != x and np.signbit(x)) else "%.17g\n" % x) for x in v.tolist()).encode()
    assert got == want
    rows = ctx.format_values(v[:1000], sep_mode=1, row=7)
    lines = rows.decode().split("\n")
    assert lines[0].split(",") == [("%.17g" % x) for x in v[:7]]
    assert len(lines) == 1000 // 7 + 1 and lines[-1].endswith(",")  # 142 rows + the open last row


GRIDS = [P.Grid.make2d(37, 11, 2.0, 1.0), P.Grid.make3d(19, 7, 5, 2.0, 1.0, 0.7),
         P.Grid.make3d(45, 9, 4, 1.0, 1.0, 1.0)]  # nx = 45: padded rows (pitch 48)


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_csv_vtk_pgm_match_reference_writers(port, tmp_path, gi):
    g = GRIDS[gi]
    comps = g.dim
    N = g.num_nodes
    state = np.concatenate([special_field(N, 20 + c) for c in range(comps)])
    E = H.random_modulus(g, 5)
    ctx = D.Context(g, 1, 0.3, D.MODE_FAST)
    ctx.set_property(E)
    ctx.set_state(state, state)
    fr = [0.3, 0.7]
    ctx.set_design(1, [1.0, 1e-6], 0.3, 3.0, 1e-6, fr, P.Weights(0.1, 3.0, 2.0, 1.5, True, -1))
    phases = H.rng(3).uniform(0.0, 1.0, 2 * N)
    phases[5] = -0.0
    ctx.set_phases(phases)
    for c in range(comps):
        ctx.write_field_csv(S, c, tmp_path / f"dev_{c}.csv")
        port.write_field_csv(g, state[c * N:(c + 1) * N], tmp_path / f"ref_{c}.csv")
        assert read(tmp_path / f"dev_{c}.csv") == read(tmp_path / f"ref_{c}.csv"), c
    names = ["phase_0", "phase_1", "modulus"] + ["displacement_" + "xyz"[c] for c in range(comps)]
    arrays = [(PH, 0, names[0]), (PH, 1, names[1]), (PR, 0, names[2])] + [(S, c, names[3 + c]) for c in range(comps)]
    ctx.write_vtk(arrays, tmp_path / "dev.vtk")
    port.write_vtk(g, [(names[0], phases[:N]), (names[1], phases[N:]), (names[2], E)]
                   + [(names[3 + c], state[c * N:(c + 1) * N]) for c in range(comps)], tmp_path / "ref.vtk")
    assert read(tmp_path / "dev.vtk") == read(tmp_path / "ref.vtk")
    if g.dim == 2:
        for c, field in ((0, S), (1, S)):
            ctx.write_pgm(field, c, tmp_path / "dev.pgm")
            port.write_pgm(g, state[c * N:(c + 1) * N], tmp_path / "ref.pgm")
            assert read(tmp_path / "dev.pgm") == read(tmp_path / "ref.pgm")
            assert read(tmp_path / "dev.pgm.scale.txt") == read(tmp_path / "ref.pgm.scale.txt")
        ctx.write_pgm(PH, 0, tmp_path / "dev.pgm")
        port.write_pgm(g, phases[:N], tmp_path / "ref.pgm")
        assert read(tmp_path / "dev.pgm") == read(tmp_path / "ref.pgm")
        assert read(tmp_path / "dev.pgm.scale.txt") == read(tmp_path / "ref.pgm.scale.txt")


def test_pgm_signed_zero_and_no_finite_values(port, tmp_path):
    g = P.Grid.make2d(9, 5, 1.0, 1.0)
    N = g.num_nodes
    for v in (np.where(np.arange(N) % 3 == 0, -0.0, 0.0), np.full(N, np.nan), np.where(np.arange(N) == 7, 2.0, np.inf)):
        ctx = D.Context(g, 0, 0.3, D.MODE_FAST)
        ctx.set_state(v, v)
        ctx.write_pgm(S, 0, tmp_path / "dev.pgm")
        port.write_pgm(g, v, tmp_path / "ref.pgm")
        assert read(tmp_path / "dev.pgm") == read(tmp_path / "ref.pgm")
        assert read(tmp_path / "dev.pgm.scale.txt") == read(tmp_path / "ref.pgm.scale.txt")


def test_multichunk_field(port, tmp_path):
    """More values than one writer chunk (8 Mi): the text of consecutive chunks joins exactly."""
    g = P.Grid.make3d(257, 256, 130, 2.0, 1.0, 0.5)  # 8.55 M nodes, padded rows
    N = g.num_nodes
    u = H.rng(4).uniform(-1e-3, 1e-3, N)
    ctx = D.Context(g, 0, 0.3, D.MODE_FAST)
    ctx.set_state(u, u)
    ctx.write_field_csv(S, 0, tmp_path / "dev.csv")
    port.write_field_csv(g, u, tmp_path / "ref.csv")
    assert read(tmp_path / "dev.csv") == read(tmp_path / "ref.csv")


def test_writer_errors(tmp_path):
    g = P.Grid.make3d(6, 5, 4, 1.0, 1.0, 1.0)
    ctx = D.Context(g, 1, 0.3, D.MODE_FAST)
    with pytest.raises(D.IoError, match="cannot open '.*missing/x.csv' for writing"):
        ctx.write_field_csv(S, 0, tmp_path / "missing" / "x.csv")
    with pytest.raises(ValueError, match="only 2D"):
        ctx.write_pgm(S, 0, tmp_path / "x.pgm")
    with pytest.raises(ValueError, match="out of range"):
        ctx.write_field_csv(S, 3, tmp_path / "x.csv")
    with pytest.raises(ValueError, match="design not set"):
        ctx.write_field_csv(PH, 0, tmp_path / "x.csv")
    slab = D.Context(g, 1, 0.3, D.MODE_FAST, k_range=(0, 2))
    with pytest.raises(ValueError, match="whole grid"):
        slab.write_field_csv(S, 0, tmp_path / "x.csv")

"""GPU: the fused 3D kernel at the full C5 size (512 x 256 x 256, 33.5 M nodes).

The small-grid parity tests pin every code path; these check the bench
configuration itself:
* the residual against the reference's own build (oracle/_ref, OpenMP) on the
  C5 grid: REPLICA bit-identical, FAST within 1e-12;
* size-independent properties of the FAST operator at C5: linearity, and the
  symmetry <V r(u), v> = <V r(v), u> of the volume-weighted residual (zero loads,
  no constraints), which holds for the assembled stiffness of the reference.
"""
import numpy as np
import pytest

from paper_2509_06971_b200 import device as D
from paper_2509_06971_b200 import problem as P

from . import helpers as H

pytestmark = pytest.mark.gpu

C5 = P.Grid.make3d(512, 256, 256, 2.0, 1.0, 1.0)


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def lumped_volume(g):
    """cell_volume (grid.hpp:64-73) per node, x-fastest."""
    ext = []
    for a in range(3):
        e = np.full(g.n[a], g.spacing[a])
        e[0] *= 0.5
        e[-1] *= 0.5
        ext.append(e)
    return (ext[2][:, None, None] * ext[1][None, :, None] * ext[0][None, None, :]).ravel()


@pytest.fixture(scope="module")
def modulus():
    return H.random_modulus(C5, 21)


def test_c5_residual_matches_reference(ref, modulus):
    g = C5
    u = H.random_field(3 * g.num_nodes, 22, -1e-3, 1e-3)
    f = H.sparse_loads(g, 3, 23, count=64)
    bc = H.elastic_bc(g, "x_hi")
    want = ref.elasticity_residual(g, bc, modulus, 0.3, f, u)
    for mode in (D.MODE_REPLICA, D.MODE_FAST):
        got = D.ElasticityOperator(g, modulus, 0.3, f, bc, mode=mode).residual(u)
        if mode == D.MODE_REPLICA:
            assert np.array_equal(got, want)
        else:
            assert rel_err(got, want) < 1e-12


def test_c5_fast_linear_and_symmetric(modulus):
    g = C5
    bc = P.BoundarySpec.all_faces(3, P.TRACTION_FREE)  # no constraints
    op = D.ElasticityOperator(g, modulus, 0.3, np.zeros(3 * g.num_nodes), bc, mode=D.MODE_FAST)
    u = H.random_field(3 * g.num_nodes, 31, -1e-3, 1e-3)
    v = H.random_field(3 * g.num_nodes, 32, -1e-3, 1e-3)
    ru, rv = op.residual(u), op.residual(v)
    a, b = 0.75, -1.25
    rw = op.residual(a * u + b * v)
    assert rel_err(rw, a * ru + b * rv) < 1e-11
    V = np.tile(lumped_volume(g), 3)
    s1, s2 = float(np.dot(V * ru, v)), float(np.dot(V * rv, u))
    assert abs(s1 - s2) <= 1e-10 * max(abs(s1), abs(s2))


def test_c5_hybrid_solve_matches_reference(ref, modulus):
    """Eight semi-implicit APT steps on the C5 grid (clamped x_hi face, sparse
    loads): REPLICA bit-identical to the reference build, FAST within 1e-10."""
    g = C5
    f = H.sparse_loads(g, 3, 41, count=64)
    bc = H.elastic_bc(g, "x_hi")
    cur = H.random_field(3 * g.num_nodes, 42, -1e-4, 1e-4)
    prev = H.random_field(3 * g.num_nodes, 43, -1e-4, 1e-4)
    h = g.min_spacing()
    p = P.PTParams(dt_pt=h * h / 8, dt_apt=0.1 * h, theta=1.0, n_apt=8, n_pt=0, form=1)
    rc, want_c, want_p, _ = ref.hybrid_solve(1, g, bc, modulus, 0.3, f, cur, prev, p)
    assert rc == 0
    for mode in (D.MODE_REPLICA, D.MODE_FAST):
        op = D.ElasticityOperator(g, modulus, 0.3, f, bc, mode=mode)
        hist = D.StateHistory(cur.copy(), prev.copy())
        D.hybrid_solve(hist, op, p)
        if mode == D.MODE_REPLICA:
            assert np.array_equal(hist.current, want_c) and np.array_equal(hist.previous, want_p)
        else:
            assert rel_err(hist.current, want_c) < 1e-10

"""Shared seeded inputs for the parity tests (SURVEY.md 8d input recipes)."""
import numpy as np

from paper_2509_06971_b200 import problem as P


def rng(seed):
    return np.random.default_rng(seed)


def random_modulus(g, seed=1, floor=1e-6):
    """E = max(floor, U^3) -- the throughput-sweep distribution."""
    u = rng(seed).random(g.num_nodes)
    return np.maximum(floor, u ** 3)


def random_field(n, seed, lo=-0.1, hi=0.1):
    return rng(seed).uniform(lo, hi, n)


def sparse_loads(g, comps, seed, count=5):
    r = rng(seed)
    f = np.zeros(comps * g.num_nodes)
    nodes = r.choice(g.num_nodes, size=min(count, g.num_nodes), replace=False)
    for n in nodes:
        for c in range(comps):
            f[c * g.num_nodes + n] = r.uniform(-1, 1)
    return f


def elastic_bc(g, clamp="x_hi", pins=()):
    bc = P.BoundarySpec.all_faces(g.dim, P.TRACTION_FREE)
    if clamp:
        bc.face[P.FACE_NAMES.index(clamp)] = P.FaceCondition(P.DIRICHLET, 0.0, 0)
    bc.pins = list(pins)
    return bc


def heat_bc(g, faces=("x_lo", "y_hi"), value=0.0):
    bc = P.BoundarySpec.all_faces(g.dim, P.NEUMANN_ZERO)
    for f in faces:
        bc.face[P.FACE_NAMES.index(f)] = P.FaceCondition(P.DIRICHLET, value, 0)
    return bc


GRIDS_2D = [(17, 9, 2.0, 1.0), (33, 20, 4.0, 1.0)]
GRIDS_3D = [(7, 6, 5, 1.0, 0.8, 0.6), (12, 9, 10, 2.0, 1.0, 1.0)]


def grids():
    out = [P.Grid.make2d(*a) for a in GRIDS_2D]
    out += [P.Grid.make3d(*a) for a in GRIDS_3D]
    return out

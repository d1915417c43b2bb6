"""Problem assembly: the reference's config -> Problem/LoopSchedule path in numpy.

Host plumbing that builds the hot path's inputs (grid, constraint set, loads,
material, targets, weights, dt schedule) exactly as the reference does, so that
bench.py and the parity tests feed the device and the oracle identical arrays.

Mirrors (file:line in /root/reference/proj):
  Grid / cell_volume / make_constraints   include/petto/grid.hpp:21-232
  ProblemConfig + presets                 include/petto/problem_config.hpp:43-105,
                                          src/problem_config.cpp:10-162
  parse_config (key = value format)       src/config_io.cpp:104-240
  nodes_in_box / effective_weights        src/engine.cpp:12-54
  build_schedule                          src/engine.cpp:56-96
  build_problem                           include/petto/engine.hpp:27-97

Pinned against the reference's own build_problem/build_schedule by
tests/test_problem.py (golden JSON under tests/golden/).
"""
from __future__ import annotations

import copy
import dataclasses
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

# CondKind order (grid.hpp:149)
DIRICHLET, NEUMANN_ZERO, TRACTION_FREE, ROLLER = 0, 1, 2, 3
FACE_NAMES = ["x_lo", "x_hi", "y_lo", "y_hi", "z_lo", "z_hi"]


class ConfigError(ValueError):
    """ConfigError (errors.hpp:28-31)."""


# --------------------------------------------------------------------- grid


class Grid:
    """Node-centred structured grid (grid.hpp:21-90)."""

    def __init__(self, dim, n, length):
        if dim not in (2, 3):
            raise ValueError("grid: dim must be 2 or 3")
        n = [int(v) for v in n] + [1] * (3 - len(n))
        length = [float(v) for v in length] + [0.0] * (3 - len(length))
        self.dim = dim
        self.n = [n[0], n[1], n[2] if dim == 3 else 1]
        self.length = [length[0], length[1], length[2] if dim == 3 else 0.0]
        self.spacing = [1.0, 1.0, 1.0]
        for a in range(dim):
            if self.n[a] < 3:
                raise ValueError("grid: need at least 3 nodes per axis")
            if not self.length[a] > 0.0:
                raise ValueError("grid: axis length must be positive")
            self.spacing[a] = self.length[a] / float(self.n[a] - 1)

    @staticmethod
    def make2d(nx, ny, lx, ly):
        return Grid(2, [nx, ny, 1], [lx, ly, 0.0])

    @staticmethod
    def make3d(nx, ny, nz, lx, ly, lz):
        return Grid(3, [nx, ny, nz], [lx, ly, lz])

    @property
    def num_nodes(self):
        return self.n[0] * self.n[1] * self.n[2]

    def node(self, i, j, k=0):
        return (k * self.n[1] + j) * self.n[0] + i

    def coord(self, axis, i):
        return self.spacing[axis] * float(i)

    def min_spacing(self):
        return min(self.spacing[: self.dim])

    def domain_volume(self):
        v = 1.0
        for a in range(self.dim):
            v *= self.length[a]
        return v

    def cell_extent(self, axis):
        """Per-index lumped extent along one axis (grid.hpp:64-67), as an array."""
        n = self.n[axis]
        if n == 1:
            return np.ones(1)
        e = np.full(n, self.spacing[axis])
        e[0] = e[-1] = 0.5 * self.spacing[axis]
        return e

    def cell_volumes(self):
        """cell_volume(i,j,k) for every node, same multiplication order as grid.hpp:69-73."""
        ex, ey, ez = self.cell_extent(0), self.cell_extent(1), self.cell_extent(2)
        v = ex[None, :] * ey[:, None]
        if self.dim == 3:
            v = v[None, :, :] * ez[:, None, None]
        else:
            v = v[None, :, :]
        return np.ascontiguousarray(v.reshape(-1))

    def ijk(self):
        k, j, i = np.meshgrid(np.arange(self.n[2]), np.arange(self.n[1]), np.arange(self.n[0]), indexing="ij")
        return i.reshape(-1), j.reshape(-1), k.reshape(-1)


@dataclass
class FaceCondition:
    kind: int = NEUMANN_ZERO
    value: float = 0.0
    component: int = 0


@dataclass
class BoundarySpec:
    """BoundarySpec (grid.hpp:169-172); pins are (node, component, value)."""

    face: List[FaceCondition] = field(default_factory=lambda: [FaceCondition() for _ in range(6)])
    pins: List[tuple] = field(default_factory=list)

    @staticmethod
    def all_faces(dim, kind, value=0.0):
        bc = BoundarySpec()
        for f in range(2 * dim):
            bc.face[f] = FaceCondition(kind, value, 0)
        return bc


def make_constraints(g: Grid, bc: BoundarySpec, comps: int):
    """make_constraints (grid.hpp:185-232): sorted entries comp*N+node, later wins."""
    nn = g.num_nodes
    has = np.zeros(nn * comps, dtype=bool)
    val = np.zeros(nn * comps)
    shape = (g.n[2], g.n[1], g.n[0])
    for f in range(2 * g.dim):
        fc = bc.face[f]
        if fc.kind not in (DIRICHLET, ROLLER):
            continue
        a = f // 2
        fixed = g.n[a] - 1 if f % 2 else 0
        mask = np.zeros(shape, dtype=bool)
        sl = [slice(None)] * 3
        sl[2 - a] = fixed
        mask[tuple(sl)] = True
        nodes = np.nonzero(mask.reshape(-1))[0]
        if fc.kind == DIRICHLET:
            for c in range(comps):
                has[c * nn + nodes] = True
                val[c * nn + nodes] = fc.value
        elif fc.component < comps:
            has[fc.component * nn + nodes] = True
            val[fc.component * nn + nodes] = fc.value
    for node, comp, value in bc.pins:
        if node < 0 or node >= nn:
            raise ValueError("boundary: pin references a node outside the grid")
        if comp < 0 or comp >= comps:
            raise ValueError("boundary: pin references an invalid component")
        has[comp * nn + node] = True
        val[comp * nn + node] = value
    entries = np.nonzero(has)[0].astype(np.int64)
    return entries, val[entries].copy()


# ------------------------------------------------------------------- config


@dataclass
class BoxSpec:
    lo: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])
    hi: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])


@dataclass
class LoadSpec:
    box: BoxSpec
    direction: List[float]
    magnitude: float


@dataclass
class RollerSpec:
    box: BoxSpec
    component: int


@dataclass
class ProblemConfig:
    """ProblemConfig (problem_config.hpp:43-105)."""

    preset: str = ""
    physics: str = "heat"  # heat | elasticity
    nx: int = 0
    ny: int = 0
    nz: int = 1
    lengths: List[float] = field(default_factory=lambda: [0.0, 0.0, 0.0])
    dirichlet_faces: List[str] = field(default_factory=list)
    dirichlet_value: float = 0.0
    fixed_faces: List[str] = field(default_factory=list)
    rollers: List[RollerSpec] = field(default_factory=list)
    loads: List[LoadSpec] = field(default_factory=list)
    source: float = 0.0
    properties: List[float] = field(default_factory=list)
    poisson_ratio: float = 0.3
    penalty: float = 3.0
    void_floor: float = 1e-6
    target_fractions: List[float] = field(default_factory=list)
    has_region: bool = False
    region_box: BoxSpec = field(default_factory=BoxSpec)
    region_fractions: List[float] = field(default_factory=list)
    alpha_compliance: float = 0.1
    alpha_volume: float = 0.0
    alpha_unity: float = 0.0
    alpha_region: float = 0.0
    normalize_compliance: bool = True
    compliance_sign: int = 1
    weight_ref_nodes: float = 0.0
    n_apt: int = 0
    n_pt: int = 0
    dt_pt: float = 0.0
    dt_apt: float = 0.0
    dt_ch: float = 0.0
    dt_ch_multiplier: float = 500.0
    theta: float = 1.0
    apt_form: str = "explicit"
    ch_mobility: float = 1.0
    ch_gamma: float = 3e-5
    max_loops: int = 1
    convergence_tol: float = 1e-3
    convergence_window: int = 50
    report_every: int = 10
    initial_phase: float = 0.5
    initial_state: float = 0.0
    # execution & output (problem_config.hpp:98-102)
    out_dir: str = ""
    precision: str = "f64"
    threads: int = 1
    formats: List[str] = field(default_factory=lambda: ["csv", "pgm", "vtk"])


def _common():
    c = ProblemConfig()
    c.alpha_compliance = 0.1
    c.normalize_compliance = True
    c.penalty = 3.0
    c.void_floor = 1e-6
    c.ch_gamma = 3e-5
    c.ch_mobility = 1.0
    c.dt_ch_multiplier = 500.0
    c.theta = 1.0
    c.convergence_tol = 1e-3
    c.convergence_window = 50
    return c


def make_preset(name: str) -> ProblemConfig:
    """The four presets (src/problem_config.cpp:28-162)."""
    c = _common()
    c.preset = name
    if name == "heat2d":
        c.physics = "heat"
        c.nx, c.ny, c.nz = 128, 128, 1
        c.lengths = [4.0, 4.0, 0.0]
        c.dirichlet_faces = ["x_lo", "y_hi"]
        c.dirichlet_value = 0.0
        c.source = 0.01
        c.properties = [1.0, 1e-6]
        c.target_fractions = [0.3, 0.7]
        c.alpha_volume, c.alpha_unity = 1e5, 1e4
        c.weight_ref_nodes = 512.0 * 512.0
        c.compliance_sign = -1
        c.n_apt, c.n_pt = 500, 500
        c.apt_form = "explicit"
        c.max_loops, c.report_every = 1200, 5
        c.initial_phase, c.initial_state = 1.0, 0.0
    elif name == "mbb2d":
        c.physics = "elasticity"
        c.nx, c.ny, c.nz = 129, 33, 1
        c.lengths = [4.0, 1.0, 0.0]
        c.properties = [1.0, 0.775, 0.55, 0.325, 0.1, 1e-6]
        c.poisson_ratio = 0.3
        c.target_fractions = [0.08, 0.08, 0.08, 0.08, 0.08, 0.6]
        c.rollers = [
            RollerSpec(BoxSpec([0.0, 0.0, 0.0], [0.0, 0.0, 0.0]), 1),
            RollerSpec(BoxSpec([4.0, 0.0, 0.0], [4.0, 0.0, 0.0]), 1),
        ]
        c.loads = [LoadSpec(BoxSpec([2.0, 1.0, 0.0], [2.0, 1.0, 0.0]), [0.0, -1.0, 0.0], 1.0)]
        c.alpha_volume, c.alpha_unity = 1e4, 1e3
        c.weight_ref_nodes = 513.0 * 128.0
        c.compliance_sign = -1
        c.n_apt, c.n_pt = 20, 20
        c.theta = 1.0
        c.apt_form = "semi_implicit"
        c.max_loops, c.report_every = 4000, 20
        c.initial_phase, c.initial_state = 0.5, 0.0
    elif name == "cantilever3d":
        c.physics = "elasticity"
        c.nx, c.ny, c.nz = 64, 9, 22
        c.lengths = [2.0, 2.0 / 15.0, 2.0 / 3.0]
        c.properties = [1.0, 0.6, 0.2, 1e-6]
        c.poisson_ratio = 0.3
        c.target_fractions = [0.1, 0.1, 0.1, 0.7]
        c.fixed_faces = ["x_hi"]
        c.loads = [LoadSpec(BoxSpec([0.0, 0.0, 1.0 / 3.0], [0.0, 2.0 / 15.0, 1.0 / 3.0]), [0.0, 0.0, 1.0], 1.0)]
        c.alpha_volume, c.alpha_unity = 1e4, 1e3
        c.weight_ref_nodes = 256.0 * 17.0 * 85.0
        c.compliance_sign = -1
        c.n_apt, c.n_pt = 100, 100
        c.theta = 1.0
        c.apt_form = "semi_implicit"
        c.max_loops, c.report_every = 500, 10
        c.initial_phase, c.initial_state = 0.5, 0.0
    elif name == "drone3d":
        c.physics = "elasticity"
        c.nx, c.ny, c.nz = 48, 24, 48
        c.lengths = [1.0, 0.5, 1.0]
        c.properties = [1.0, 1e-6]
        c.poisson_ratio = 0.3
        c.target_fractions = [0.2, 0.8]
        s = math.cbrt(0.2)  # std::cbrt, same libm
        c.region_box = BoxSpec([0.5 * c.lengths[a] * (1.0 - s) for a in range(3)],
                               [0.5 * c.lengths[a] * (1.0 + s) for a in range(3)])
        c.has_region = True
        c.region_fractions = [0.0, 1.0]
        c.rollers = [
            RollerSpec(BoxSpec([0.0, 0.5, 0.0], [0.0, 0.5, 0.0]), 1),
            RollerSpec(BoxSpec([1.0, 0.5, 0.0], [1.0, 0.5, 0.0]), 1),
            RollerSpec(BoxSpec([0.0, 0.5, 1.0], [0.0, 0.5, 1.0]), 1),
            RollerSpec(BoxSpec([1.0, 0.5, 1.0], [1.0, 0.5, 1.0]), 1),
        ]
        c.loads = [LoadSpec(BoxSpec([0.5, 0.0, 0.5], [0.5, 0.0, 0.5]), [0.0, -1.0, 0.0], 1.0)]
        c.alpha_volume, c.alpha_unity, c.alpha_region = 1e4, 1e3, 1e4
        c.weight_ref_nodes = 128.0 * 64.0 * 128.0
        c.compliance_sign = -1
        c.n_apt, c.n_pt = 50, 50
        c.theta = 1.0
        c.apt_form = "semi_implicit"
        c.max_loops, c.report_every = 800, 10
        c.initial_phase, c.initial_state = 0.5, 0.0
    else:
        raise ConfigError(f"unknown preset '{name}'; valid presets: heat2d mbb2d cantilever3d drone3d")
    return c


def _parse_double(key, v):
    try:
        return float(v)
    except ValueError:
        raise ConfigError(f"config field '{key}': cannot parse number '{v}'") from None


def _split_list(v):
    return [s.strip() for s in v.split(",") if s.strip()]


def _parse_box(key, v):
    nums = [_parse_double(key, s) for s in _split_list(v)]
    if len(nums) != 6:
        raise ConfigError(f"config field '{key}': box needs 6 numbers (x0,y0,z0,x1,y1,z1)")
    return BoxSpec(nums[:3], nums[3:])


def _component(name):
    return {"x": 0, "0": 0, "y": 1, "1": 1, "z": 2, "2": 2}[name]


def parse_config(text: str) -> ProblemConfig:
    """parse_config (src/config_io.cpp:206-240) for the key = value format."""
    entries, preset = [], ""
    for lineno, line in enumerate(text.splitlines(), 1):
        s = line.strip()
        if "#" in s:
            s = s[: s.index("#")].strip()
        if not s or s.startswith("["):
            continue
        if "=" not in s:
            raise ConfigError(f"<text>:{lineno}: expected 'key = value'")
        k, v = s.split("=", 1)
        k, v = k.strip(), v.strip()
        if k == "preset":
            preset = v
        else:
            entries.append((k, v, lineno))
    c = make_preset(preset) if preset else ProblemConfig()
    if not preset:
        c.preset = ""
    deferred = {}
    plain_float = {"dirichlet_value", "source", "poisson_ratio", "penalty", "void_floor", "alpha_compliance",
                   "alpha_volume", "alpha_unity", "alpha_region", "weight_ref_nodes", "dt_pt", "dt_apt", "dt_ch",
                   "dt_ch_multiplier", "theta", "ch_mobility", "ch_gamma", "convergence_tol", "initial_phase",
                   "initial_state"}
    plain_int = {"nx", "ny", "nz", "n_apt", "n_pt", "max_loops", "convergence_window", "report_every",
                 "compliance_sign"}
    for k, v, lineno in entries:
        if k == "physics":
            if v not in ("heat", "elasticity"):
                raise ConfigError("config field 'physics': must be 'heat' or 'elasticity'")
            c.physics = v
        elif k in plain_int:
            setattr(c, k, int(_parse_double(k, v)))
        elif k in plain_float:
            setattr(c, k, _parse_double(k, v))
        elif k in ("length_x", "length_y", "length_z"):
            c.lengths["xyz".index(k[-1])] = _parse_double(k, v)
        elif k in ("dirichlet_faces", "fixed_faces"):
            setattr(c, k, _split_list(v))
        elif k in ("properties", "target_fractions"):
            setattr(c, k, [_parse_double(k, s) for s in _split_list(v)])
        elif k == "region_box":
            c.region_box = _parse_box(k, v)
            c.has_region = True
        elif k == "region_fractions":
            c.region_fractions = [_parse_double(k, s) for s in _split_list(v)]
            c.has_region = bool(c.region_fractions)
        elif k == "normalize_compliance":
            c.normalize_compliance = v in ("true", "on", "1")
        elif k == "apt_form":
            c.apt_form = v
        elif k.startswith("roller_") or k.startswith("load_") or k in ("roller_count", "load_count"):
            deferred[k] = v
        elif k in ("out_dir", "precision"):
            setattr(c, k, v)
        elif k == "threads":
            c.threads = int(_parse_double(k, v))
        elif k == "formats":
            c.formats = _split_list(v)
        else:
            raise ConfigError(f"line {lineno}: unknown config key '{k}'")
    if "roller_count" in deferred:
        c.rollers = []
        for i in range(int(_parse_double("roller_count", deferred["roller_count"]))):
            b = f"roller_{i}"
            c.rollers.append(RollerSpec(_parse_box(b + "_box", deferred[b + "_box"]),
                                        _component(deferred[b + "_component"])))
    if "load_count" in deferred:
        c.loads = []
        for i in range(int(_parse_double("load_count", deferred["load_count"]))):
            b = f"load_{i}"
            d = [_parse_double(b, s) for s in _split_list(deferred[b + "_direction"])]
            c.loads.append(LoadSpec(_parse_box(b + "_box", deferred[b + "_box"]), d,
                                    _parse_double(b, deferred[b + "_magnitude"])))
    return c


def validate_config(c: ProblemConfig):
    """validate_config (src/problem_config.cpp:219-299): ConfigError on the first violation."""
    def fail(fld, constraint):
        raise ConfigError(f"config field '{fld}': {constraint}")

    def check_box(fld, b, dim):
        for a in range(dim):
            if b.lo[a] > b.hi[a]:
                fail(fld, "box lo must not exceed hi")
            if b.lo[a] < -1e-9 or b.hi[a] > c.lengths[a] + 1e-9:
                fail(fld, "box must lie inside the domain")

    dim = 3 if c.nz > 1 else 2
    if c.nx < 3:
        fail("nx", "needs at least 3 nodes per axis")
    if c.ny < 3:
        fail("ny", "needs at least 3 nodes per axis")
    if dim == 3 and c.nz < 3:
        fail("nz", "needs at least 3 nodes per axis (or 1 for 2D)")
    for a in range(dim):
        if not c.lengths[a] > 0.0:
            fail("lengths", "domain extents must be positive")
    if not c.properties:
        fail("properties", "at least one phase property required")
    if any(not p > 0.0 for p in c.properties):
        fail("properties", "must be positive")
    if c.penalty < 1.0:
        fail("penalty", "must be >= 1")
    if not c.void_floor > 0.0:
        fail("void_floor", "must be positive")
    if c.physics == "elasticity" and (c.poisson_ratio <= -1.0 or c.poisson_ratio >= 0.5):
        fail("poisson_ratio", "must lie in (-1, 0.5)")
    if len(c.target_fractions) != len(c.properties):
        fail("target_fractions", "one target per phase required")
    total = 0.0
    for t in c.target_fractions:
        if t < 0.0 or t > 1.0:
            fail("target_fractions", "each target must lie in [0,1]")
        total += t
    if total > 1.0 + 1e-6:
        fail("target_fractions", "targets must sum to at most 1")
    if c.has_region:
        if len(c.region_fractions) != len(c.properties):
            fail("region_fractions", "one region target per phase required")
        if any(t < 0.0 or t > 1.0 for t in c.region_fractions):
            fail("region_fractions", "targets must lie in [0,1]")
        check_box("region_box", c.region_box, dim)
    if min(c.alpha_compliance, c.alpha_volume, c.alpha_unity, c.alpha_region) < 0:
        fail("alpha_*", "weights must be non-negative")
    if c.alpha_compliance + c.alpha_volume + c.alpha_unity + c.alpha_region <= 0:
        fail("alpha_*", "at least one weight must be positive")
    if c.compliance_sign not in (1, -1):
        fail("compliance_sign", "must be +1 or -1")
    if c.weight_ref_nodes < 0:
        fail("weight_ref_nodes", "must be >= 0")
    if c.n_apt < 0 or c.n_pt < 0 or c.n_apt + c.n_pt < 1:
        fail("n_apt/n_pt", "need at least one state step per loop")
    if not c.theta > 0.0:
        fail("theta", "must be positive")
    if c.apt_form not in ("explicit", "semi_implicit"):
        fail("apt_form", "must be 'explicit' or 'semi_implicit'")
    if not c.ch_mobility > 0.0:
        fail("ch_mobility", "must be positive")
    if not c.ch_gamma > 0.0:
        fail("ch_gamma", "must be positive")
    if c.dt_pt < 0 or c.dt_apt < 0 or c.dt_ch < 0:
        fail("dt_*", "must be >= 0 (0 = auto)")
    if c.dt_ch == 0.0 and not c.dt_ch_multiplier > 0.0:
        fail("dt_ch_multiplier", "must be positive when dt_ch is auto")
    if c.max_loops < 1:
        fail("max_loops", "must be >= 1")
    if not c.convergence_tol > 0.0:
        fail("convergence_tol", "must be positive")
    if c.convergence_window < 2:
        fail("convergence_window", "must be >= 2")
    if c.report_every < 1:
        fail("report_every", "must be >= 1")
    faces = FACE_NAMES[: 2 * dim]
    if c.physics == "heat":
        if any(f not in faces for f in c.dirichlet_faces):
            fail("dirichlet_faces", "face not in domain")
    else:
        if any(f not in faces for f in c.fixed_faces):
            fail("fixed_faces", "face not in domain")
        for r in c.rollers:
            check_box("rollers", r.box, dim)
            if r.component < 0 or r.component >= dim:
                fail("rollers", "invalid component")
        for ld in c.loads:
            check_box("loads", ld.box, dim)
            if not sum(d * d for d in ld.direction) > 0.0:
                fail("loads", "direction must be nonzero")
    if c.precision not in ("f32", "f64"):
        fail("precision", "must be 'f32' or 'f64'")
    if c.threads < 0:
        fail("threads", "must be >= 0")
    if c.initial_phase < 0.0 or c.initial_phase > 1.0:
        fail("initial_phase", "must lie in [0,1]")


# --------------------------------------------------------------- assembly


def make_grid(cfg: ProblemConfig) -> Grid:
    """make_grid (src/engine.cpp:32-37)."""
    if cfg.nz > 1:
        return Grid.make3d(cfg.nx, cfg.ny, cfg.nz, *cfg.lengths)
    return Grid.make2d(cfg.nx, cfg.ny, cfg.lengths[0], cfg.lengths[1])


def nodes_in_box(g: Grid, box: BoxSpec):
    """nodes_in_box (src/engine.cpp:12-30), ascending node order."""
    inside = np.ones(g.num_nodes, dtype=bool)
    idx = g.ijk()
    for a in range(g.dim):
        x = g.spacing[a] * idx[a].astype(np.float64)
        tol = 0.5 * g.spacing[a] * (1.0 + 1e-9)
        inside &= ~((x < box.lo[a] - tol) | (x > box.hi[a] + tol))
    return np.nonzero(inside)[0].astype(np.int64)


@dataclass
class Weights:
    alpha_compliance: float = 0.1
    alpha_volume: float = 0.0
    alpha_unity: float = 0.0
    alpha_region: float = 0.0
    normalize_compliance: bool = True
    compliance_sign: int = 1


def effective_weights(cfg: ProblemConfig, g: Grid) -> Weights:
    """effective_weights (src/engine.cpp:39-54)."""
    w = Weights(cfg.alpha_compliance, cfg.alpha_volume, cfg.alpha_unity, cfg.alpha_region,
                cfg.normalize_compliance, cfg.compliance_sign)
    if cfg.weight_ref_nodes > 0.0:
        scale = float(g.num_nodes) / cfg.weight_ref_nodes
        w.alpha_volume *= scale
        w.alpha_region *= scale
        w.alpha_unity *= scale / g.domain_volume()
    return w


@dataclass
class PTParams:
    dt_pt: float = 0.0
    dt_apt: float = 0.0
    theta: float = 1.0
    n_apt: int = 0
    n_pt: int = 0
    form: int = 0  # 0 explicit, 1 semi-implicit


@dataclass
class Schedule:
    pt: PTParams
    ch_mobility: float = 1.0
    ch_gamma: float = 3e-5
    dt_ch: float = 0.0
    max_loops: int = 1
    convergence_tol: float = 1e-3
    convergence_window: int = 50
    report_every: int = 1


def ch_stable_dt(g: Grid, mobility, gamma):
    """ch_stable_dt (phase_field.hpp:26-31)."""
    s = 0.0
    for a in range(g.dim):
        s += 4.0 / (g.spacing[a] * g.spacing[a])
    wpp_max = math.pi * math.pi / 32.0
    return 2.0 / (mobility * (gamma * s * s + wpp_max * s))


def build_schedule(cfg: ProblemConfig, g: Grid, spectral_bound=None) -> Schedule:
    """build_schedule (src/engine.cpp:56-96).

    spectral_bound(g, nu, e_max) must be elasticity_spectral_bound; the product's
    implementation is paper_2509_06971_b200.device.spectral_bound.
    """
    prop_max = max(cfg.properties) if cfg.properties else 0.0
    prop_max = max(prop_max, 0.0)
    prop_sum = 0.0
    for p in cfg.properties:
        prop_sum += p
    coeff = max(1.0, prop_max)
    h = g.min_spacing()
    pt = PTParams()
    pt.dt_pt = cfg.dt_pt if cfg.dt_pt > 0 else h * h / (2.0 * g.dim * coeff)
    pt.dt_apt = cfg.dt_apt if cfg.dt_apt > 0 else 0.5 * h / math.sqrt(coeff)
    if cfg.physics == "elasticity":
        if spectral_bound is None:
            from . import device

            spectral_bound = device.spectral_bound
        bound = spectral_bound(g, cfg.poisson_ratio, max(1e-300, prop_sum))
        if cfg.dt_pt <= 0:
            pt.dt_pt = min(pt.dt_pt, 0.9 * 2.0 / bound)
        if cfg.dt_apt <= 0:
            pt.dt_apt = min(pt.dt_apt, 0.9 * 2.0 / math.sqrt(bound))
    pt.theta = cfg.theta
    pt.n_apt = cfg.n_apt
    pt.n_pt = cfg.n_pt
    pt.form = 1 if cfg.apt_form == "semi_implicit" else 0
    s = Schedule(pt)
    s.ch_mobility = cfg.ch_mobility
    s.ch_gamma = cfg.ch_gamma
    if cfg.dt_ch > 0:
        s.dt_ch = cfg.dt_ch
    else:
        nominal = cfg.dt_ch_multiplier * h * h * h * h
        cap = 0.9 * ch_stable_dt(g, cfg.ch_mobility, cfg.ch_gamma)
        s.dt_ch = min(nominal, cap)
    s.max_loops = cfg.max_loops
    s.convergence_tol = cfg.convergence_tol
    s.convergence_window = cfg.convergence_window
    s.report_every = cfg.report_every
    return s


@dataclass
class Problem:
    """Problem<Real> (optimizer.hpp:66-77) plus its constraint set."""

    grid: Grid
    physics: int  # 0 heat, 1 elasticity
    bc: BoundarySpec
    properties: List[float]
    poisson_ratio: float
    penalty: float
    void_floor: float
    fractions: List[float]
    region_nodes: np.ndarray
    region_fractions: Optional[List[float]]
    weights: Weights
    source: np.ndarray  # comps x N
    initial_phases: np.ndarray  # P x N
    initial_state: np.ndarray  # comps x N
    cons_entry: np.ndarray
    cons_value: np.ndarray

    @property
    def comps(self):
        return self.grid.dim if self.physics else 1

    @property
    def nphases(self):
        return len(self.properties)

    @property
    def has_region(self):
        return self.region_fractions is not None


def build_problem(cfg: ProblemConfig) -> Problem:
    """build_problem (engine.hpp:27-97)."""
    g = make_grid(cfg)
    dim = g.dim
    nn = g.num_nodes
    bc = BoundarySpec()
    if cfg.physics == "heat":
        for f in range(2 * dim):
            bc.face[f] = FaceCondition(NEUMANN_ZERO, 0.0, 0)
        for name in cfg.dirichlet_faces:
            bc.face[FACE_NAMES.index(name)] = FaceCondition(DIRICHLET, cfg.dirichlet_value, 0)
        source = np.full(nn, float(cfg.source))
        comps = 1
    else:
        for f in range(2 * dim):
            bc.face[f] = FaceCondition(TRACTION_FREE, 0.0, 0)
        for name in cfg.fixed_faces:
            bc.face[FACE_NAMES.index(name)] = FaceCondition(DIRICHLET, 0.0, 0)
        for r in cfg.rollers:
            for node in nodes_in_box(g, r.box):
                bc.pins.append((int(node), r.component, 0.0))
        comps = dim
        source = np.zeros(dim * nn)
        for load in cfg.loads:
            nodes = nodes_in_box(g, load.box)
            if len(nodes) == 0:
                raise ConfigError("config field 'loads': box selects no nodes")
            norm = 0.0
            for d in load.direction:
                norm += d * d
            norm = math.sqrt(norm)
            cv = g.cell_volumes()
            lumped = 0.0
            for node in nodes:
                lumped += float(cv[node])
            for node in nodes:
                for c in range(dim):
                    source[c * nn + node] += -load.direction[c] / norm * load.magnitude / lumped
    region_nodes = np.zeros(0, np.int64)
    region_fractions = None
    if cfg.has_region:
        region_nodes = nodes_in_box(g, cfg.region_box)
        if len(region_nodes) == 0:
            raise ConfigError("config field 'region_box': selects no nodes")
        region_fractions = list(cfg.region_fractions)
    P = len(cfg.properties)
    phases = np.full(P * nn, float(cfg.initial_phase))
    state = np.full(comps * nn, float(cfg.initial_state))
    entries, values = make_constraints(g, bc, comps)
    state[entries] = values
    return Problem(g, 0 if cfg.physics == "heat" else 1, bc, list(cfg.properties), cfg.poisson_ratio,
                   cfg.penalty, cfg.void_floor, list(cfg.target_fractions), region_nodes, region_fractions,
                   effective_weights(cfg, g), source, phases, state, entries, values)


# The synthetic workloads of BASELINE.json.
CONFIGS = {
    "C1": """preset = mbb2d
nx = 160
ny = 80
length_x = 2
length_y = 1
properties = 1, 1e-6
target_fractions = 0.4, 0.6
roller_count = 0
fixed_faces = x_lo
load_count = 1
load_0_box = 2,0.5,0,2,0.5,0
load_0_direction = 0,-1,0
load_0_magnitude = 1
""",
    "C2": """preset = heat2d
nx = 256
ny = 256
""",
    "C3": """preset = mbb2d
nx = 512
ny = 256
properties = 1, 0.55, 1e-6
target_fractions = 0.2, 0.2, 0.6
""",
    "C4": """preset = cantilever3d
nx = 128
ny = 64
nz = 64
length_x = 2
length_y = 1
length_z = 1
properties = 1, 1e-6
target_fractions = 0.3, 0.7
load_count = 1
load_0_box = 0,0,0.5,0,1,0.5
load_0_direction = 0,0,1
load_0_magnitude = 1
""",
}
CONFIGS["C5"] = CONFIGS["C4"].replace("nx = 128", "nx = 512").replace("ny = 64", "ny = 256").replace(
    "nz = 64", "nz = 256")

CONFIG_NAMES = {
    "C1": "2D cantilever compliance 160x80, single material, FP64",
    "C2": "2D heat-sink thermal compliance 256x256, single material",
    "C3": "2D 3-phase MBB beam 512x256, phase-field interpolation",
    "C4": "3D cantilever elasticity 128x64x64, single material",
    "C5": "3D cantilever elasticity 512x256x256, single material",
}


def config(name: str, **overrides) -> ProblemConfig:
    cfg = parse_config(CONFIGS[name])
    for k, v in overrides.items():
        setattr(cfg, k, v)
    return cfg

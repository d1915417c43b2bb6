"""ctypes binding of oracle/petto_oracle.h -- TEST INFRASTRUCTURE ONLY.

Loads either implementation of the oracle interface:

* ``load("port")``      -> oracle/liboracle.so        (plain-C restatement)
* ``load("reference")`` -> oracle/_ref/libpetto_ref.so (the reference itself)

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libpetto_ref.so")

MAX_PHASES = 8


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int), ("n", C.c_int64 * 3), ("length", C.c_double * 3)]


class BC(C.Structure):
    _fields_ = [
        ("kind", C.c_int * 6),
        ("value", C.c_double * 6),
        ("component", C.c_int * 6),
        ("npins", C.c_int64),
        ("pin_node", C.POINTER(C.c_int64)),
        ("pin_comp", C.POINTER(C.c_int32)),
        ("pin_value", C.POINTER(C.c_double)),
    ]


class PTParams(C.Structure):
    _fields_ = [
        ("dt_pt", C.c_double),
        ("dt_apt", C.c_double),
        ("theta", C.c_double),
        ("n_apt", C.c_long),
        ("n_pt", C.c_long),
        ("form", C.c_int),
    ]


class SolveStats(C.Structure):
    _fields_ = [
        ("iterations", C.c_long),
        ("r_initial", C.c_double),
        ("r_final", C.c_double),
        ("converged", C.c_int),
    ]


class Material(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("nphases", C.c_int),
        ("properties", C.POINTER(C.c_double)),
        ("poisson_ratio", C.c_double),
        ("penalty", C.c_double),
        ("void_floor", C.c_double),
    ]


class Targets(C.Structure):
    _fields_ = [
        ("fractions", C.POINTER(C.c_double)),
        ("nregion", C.c_int64),
        ("region_nodes", C.POINTER(C.c_int64)),
        ("region_fractions", C.POINTER(C.c_double)),
    ]


class Weights(C.Structure):
    _fields_ = [
        ("alpha_compliance", C.c_double),
        ("alpha_volume", C.c_double),
        ("alpha_unity", C.c_double),
        ("alpha_region", C.c_double),
        ("normalize_compliance", C.c_int),
        ("compliance_sign", C.c_int),
    ]


class CHParams(C.Structure):
    _fields_ = [("mobility", C.c_double), ("gamma", C.c_double), ("dt", C.c_double)]


class CHStats(C.Structure):
    _fields_ = [("mass_before", C.c_double), ("mass_preclamp", C.c_double), ("mass_postclamp", C.c_double)]


class Report(C.Structure):
    _fields_ = [
        ("compliance", C.c_double),
        ("volume", C.c_double),
        ("unity", C.c_double),
        ("region", C.c_double),
        ("volume_fractions", C.c_double * MAX_PHASES),
    ]


class Problem(C.Structure):
    _fields_ = [
        ("grid", Grid),
        ("physics", C.c_int),
        ("bc", BC),
        ("material", Material),
        ("targets", Targets),
        ("weights", Weights),
        ("source", C.POINTER(C.c_double)),
        ("initial_phases", C.POINTER(C.c_double)),
        ("initial_state", C.POINTER(C.c_double)),
    ]


class Schedule(C.Structure):
    _fields_ = [
        ("pt", PTParams),
        ("ch", CHParams),
        ("max_loops", C.c_long),
        ("convergence_tol", C.c_double),
        ("convergence_window", C.c_int),
        ("report_every", C.c_int),
    ]


class Record(C.Structure):
    _fields_ = [
        ("loop", C.c_long),
        ("apt_steps", C.c_longlong),
        ("pt_steps", C.c_longlong),
        ("compliance", C.c_double),
        ("volume", C.c_double),
        ("unity", C.c_double),
        ("region", C.c_double),
        ("r_pde", C.c_double),
        ("separation", C.c_double),
        ("volume_fractions", C.c_double * MAX_PHASES),
    ]


class RunResult(C.Structure):
    _fields_ = [
        ("loops", C.c_long),
        ("apt_steps", C.c_longlong),
        ("pt_steps", C.c_longlong),
        ("design_updates", C.c_longlong),
        ("ch_steps", C.c_longlong),
        ("clamp_mass_drift", C.c_double),
        ("termination", C.c_int),
        ("abort_detail", C.c_char * 256),
    ]


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


class _Keep:
    """Holds numpy arrays referenced by a ctypes struct."""

    def __init__(self, c, *arrays):
        self.c = c
        self.arrays = arrays


def grid_struct(g):
    """problem.Grid -> orc_grid."""
    return _Keep(Grid(g.dim, (C.c_int64 * 3)(*g.n), (C.c_double * 3)(*g.length)))


def bc_struct(bc):
    """problem.BoundarySpec -> orc_bc."""
    nodes = np.array([p[0] for p in bc.pins] or [0], dtype=np.int64)
    comps = np.array([p[1] for p in bc.pins] or [0], dtype=np.int32)
    vals = np.array([p[2] for p in bc.pins] or [0.0], dtype=np.float64)
    c = BC((C.c_int * 6)(*[f.kind for f in bc.face]), (C.c_double * 6)(*[f.value for f in bc.face]),
           (C.c_int * 6)(*[f.component for f in bc.face]), len(bc.pins),
           nodes.ctypes.data_as(C.POINTER(C.c_int64)), comps.ctypes.data_as(C.POINTER(C.c_int32)), _dp(vals))
    return _Keep(c, nodes, comps, vals)


def material_struct(kind, properties, poisson_ratio=0.3, penalty=3.0, void_floor=1e-6):
    props = np.array(properties, dtype=np.float64)
    return _Keep(Material(kind, len(props), _dp(props), poisson_ratio, penalty, void_floor), props)


def targets_struct(fractions, region_nodes=None, region_fractions=None):
    fr = np.array(fractions, dtype=np.float64)
    rn = np.array(region_nodes if region_nodes is not None else [0], dtype=np.int64)
    rf = np.array(region_fractions, dtype=np.float64) if region_fractions is not None else None
    c = Targets(_dp(fr), len(region_nodes) if region_nodes is not None else 0,
                rn.ctypes.data_as(C.POINTER(C.c_int64)), _dp(rf))
    return _Keep(c, fr, rn, rf)


def weights_struct(w):
    return Weights(w.alpha_compliance, w.alpha_volume, w.alpha_unity, w.alpha_region,
                   1 if w.normalize_compliance else 0, int(w.compliance_sign))


def pt_struct(pt):
    return PTParams(pt.dt_pt, pt.dt_apt, pt.theta, pt.n_apt, pt.n_pt, pt.form)


def schedule_struct(s):
    return Schedule(pt_struct(s.pt), CHParams(s.ch_mobility, s.ch_gamma, s.dt_ch), s.max_loops,
                    s.convergence_tol, s.convergence_window, s.report_every)


def problem_struct(prob):
    """problem.Problem -> orc_problem (plus the keep-alive list)."""
    g = grid_struct(prob.grid)
    b = bc_struct(prob.bc)
    m = material_struct(prob.physics, prob.properties, prob.poisson_ratio, prob.penalty, prob.void_floor)
    t = targets_struct(prob.fractions, prob.region_nodes if prob.has_region else None, prob.region_fractions)
    src = np.ascontiguousarray(prob.source, dtype=np.float64)
    ph = np.ascontiguousarray(prob.initial_phases, dtype=np.float64)
    st = np.ascontiguousarray(prob.initial_state, dtype=np.float64)
    c = Problem(g.c, prob.physics, b.c, m.c, t.c, weights_struct(prob.weights), _dp(src), _dp(ph), _dp(st))
    return _Keep(c, g, b, m, t, src, ph, st)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def build_port():
    """Compile the C restatement if it is missing (gcc is on every box)."""
    if not os.path.exists(PORT_LIB):
        subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    return PORT_LIB


class Oracle:
    """Python face of one oracle implementation (port or reference)."""

    def __init__(self, path):
        self.path = path
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_impl_name.restype = C.c_char_p
        L.orc_residual_norm.restype = C.c_double
        L.orc_residual_norm.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int]
        L.orc_make_constraints.restype = C.c_int64
        L.orc_elasticity_spectral_bound.restype = C.c_double
        L.orc_ch_stable_dt.restype = C.c_double
        L.orc_phase_mass.restype = C.c_double
        L.orc_gl_energy.restype = C.c_double
        L.orc_separation.restype = C.c_double
        L.orc_spacing.restype = C.c_double
        L.orc_cell_volume.restype = C.c_double
        self.name = L.orc_impl_name().decode()

    # -- helpers ----------------------------------------------------------
    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    def set_threads(self, n):
        self.lib.orc_set_threads(C.c_int(n))

    # -- a1-a12 -------------------------------------------------------------
    def make_constraints(self, grid, bc, comps):
        grid, bc = grid_struct(grid), bc_struct(bc)
        n = self.lib.orc_make_constraints(C.byref(grid.c), C.byref(bc.c), comps, None, None, 0)
        if n < 0:
            raise OracleError(int(-1 - n), self.lib.orc_last_error().decode())
        e = np.zeros(max(n, 1), np.int64)
        v = np.zeros(max(n, 1))
        self.lib.orc_make_constraints(C.byref(grid.c), C.byref(bc.c), comps,
                                      e.ctypes.data_as(C.POINTER(C.c_int64)), _dp(v), n)
        return e[:n], v[:n]

    def unit_cell_stiffness(self, dim, h, nu):
        n = (1 << dim) * dim
        out = np.zeros(n * n)
        self.lib.orc_unit_cell_stiffness(dim, (C.c_double * 3)(*h), C.c_double(nu), _dp(out))
        return out.reshape(n, n)

    def spectral_bound(self, grid, nu, emax):
        grid = grid_struct(grid)
        return self.lib.orc_elasticity_spectral_bound(C.byref(grid.c), C.c_double(nu), C.c_double(emax))

    def ch_stable_dt(self, grid, mobility, gamma):
        grid = grid_struct(grid)
        return self.lib.orc_ch_stable_dt(C.byref(grid.c), C.c_double(mobility), C.c_double(gamma))

    def heat_residual(self, grid, bc, kappa, source, T):
        out = np.zeros(grid.num_nodes)
        grid, bc = grid_struct(grid), bc_struct(bc)
        self._check(self.lib.orc_heat_residual(C.byref(grid.c), C.byref(bc.c), _dp(kappa), _dp(source),
                                               _dp(T), _dp(out)))
        return out

    def elasticity_residual(self, grid, bc, modulus, nu, loads, u):
        out = np.zeros(grid.num_nodes * grid.dim)
        grid, bc = grid_struct(grid), bc_struct(bc)
        self._check(self.lib.orc_elasticity_residual(C.byref(grid.c), C.byref(bc.c), _dp(modulus),
                                                     C.c_double(nu), _dp(loads), _dp(u), _dp(out)))
        return out

    def residual_norm(self, r, nodes, comps):
        r = np.ascontiguousarray(r, dtype=np.float64)
        return self.lib.orc_residual_norm(_dp(r), nodes, comps)

    # -- a13-a17 ------------------------------------------------------------
    def hybrid_solve(self, physics, grid, bc, prop, nu, source, cur, prev, params):
        grid, bc, params = grid_struct(grid), bc_struct(bc), pt_struct(params)
        cur = np.array(cur, dtype=np.float64, copy=True)
        prev = np.array(prev, dtype=np.float64, copy=True)
        step = C.c_int64(0)
        rc = self.lib.orc_hybrid_solve(physics, C.byref(grid.c), C.byref(bc.c), _dp(prop), C.c_double(nu),
                                       _dp(source), _dp(cur), _dp(prev), C.byref(params), C.byref(step))
        return rc, cur, prev, step.value

    def time_hybrid(self, physics, grid, bc, prop, nu, source, cur, prev, params):
        """Seconds spent inside hybrid_solve alone (operator set-up excluded)."""
        grid, bc, params = grid_struct(grid), bc_struct(bc), pt_struct(params)
        cur = np.array(cur, dtype=np.float64, copy=True)
        prev = np.array(prev, dtype=np.float64, copy=True)
        sec = C.c_double(0.0)
        self._check(self.lib.orc_time_hybrid(physics, C.byref(grid.c), C.byref(bc.c), _dp(prop), C.c_double(nu),
                                             _dp(source), _dp(cur), _dp(prev), C.byref(params), C.byref(sec)))
        return sec.value

    def iterate_to_tolerance(self, physics, grid, bc, prop, nu, source, cur, prev, mode, params,
                             target, max_iters):
        grid, bc, params = grid_struct(grid), bc_struct(bc), pt_struct(params)
        cur = np.array(cur, dtype=np.float64, copy=True)
        prev = np.array(prev, dtype=np.float64, copy=True)
        st = SolveStats()
        rc = self.lib.orc_iterate_to_tolerance(physics, C.byref(grid.c), C.byref(bc.c), _dp(prop),
                                               C.c_double(nu), _dp(source), _dp(cur), _dp(prev), mode,
                                               C.byref(params), C.c_double(target), C.c_long(max_iters),
                                               C.byref(st))
        return rc, st, cur, prev

    # -- a19-a26 ------------------------------------------------------------
    def interpolate(self, grid, mat, phases):
        out = np.zeros(grid.num_nodes)
        grid = grid_struct(grid)
        self._check(self.lib.orc_interpolate(C.byref(grid.c), C.byref(mat.c), _dp(phases), _dp(out)))
        return out

    def sensitivities(self, grid, mat, targets, phases, state):
        P, N = mat.c.nphases, grid.num_nodes
        gc, gv, gu = np.zeros(P * N), np.zeros(P * N), np.zeros(P * N)
        gr = np.zeros(P * N) if targets.c.region_fractions else None
        grid = grid_struct(grid)
        self._check(self.lib.orc_sensitivities(C.byref(grid.c), C.byref(mat.c), C.byref(targets.c),
                                               _dp(phases), _dp(state), _dp(gc), _dp(gv), _dp(gu), _dp(gr)))
        return gc, gv, gu, gr

    def design_update(self, grid, nphases, weights, phases, gc, gv, gu, gr):
        phases = np.array(phases, dtype=np.float64, copy=True)
        grid, weights = grid_struct(grid), weights_struct(weights)
        self._check(self.lib.orc_design_update(C.byref(grid.c), nphases, C.byref(weights), _dp(phases),
                                               _dp(gc), _dp(gv), _dp(gu), _dp(gr)))
        return phases

    def ch_step(self, grid, mobility, gamma, dt, phi):
        phi = np.array(phi, dtype=np.float64, copy=True)
        grid = grid_struct(grid)
        st = CHStats()
        self._check(self.lib.orc_ch_step(C.byref(grid.c), C.byref(CHParams(mobility, gamma, dt)), _dp(phi),
                                         C.byref(st)))
        return phi, (st.mass_before, st.mass_preclamp, st.mass_postclamp)

    def phase_mass(self, grid, phi):
        grid = grid_struct(grid)
        return self.lib.orc_phase_mass(C.byref(grid.c), _dp(np.ascontiguousarray(phi, dtype=np.float64)))

    def gl_energy(self, grid, phi, gamma):
        grid = grid_struct(grid)
        return self.lib.orc_gl_energy(C.byref(grid.c), _dp(np.ascontiguousarray(phi, dtype=np.float64)),
                                      C.c_double(gamma))

    def separation(self, grid, nphases, phases):
        grid = grid_struct(grid)
        return self.lib.orc_separation(C.byref(grid.c), nphases, _dp(phases))

    def evaluate_objectives(self, grid, mat, targets, phases, state):
        rep = Report()
        grid = grid_struct(grid)
        self._check(self.lib.orc_evaluate_objectives(C.byref(grid.c), C.byref(mat.c), C.byref(targets.c),
                                                     _dp(phases), _dp(state), C.byref(rep)))
        return rep

    def run(self, prob, sched, records_cap=100000):
        """prob: a paper_2509_06971_b200.problem.Problem; sched: its Schedule."""
        P, N, comps = prob.nphases, prob.grid.num_nodes, prob.comps
        phases = np.zeros(P * N)
        state = np.zeros(comps * N)
        recs = (Record * records_cap)()
        nrec = C.c_long(0)
        res = RunResult()
        keep = problem_struct(prob)
        self._check(self.lib.orc_run(C.byref(keep.c), C.byref(schedule_struct(sched)), _dp(phases), _dp(state),
                                     recs, records_cap, C.byref(nrec), C.byref(res)))
        return phases, state, [recs[i] for i in range(min(nrec.value, records_cap))], res

    # -- output writers (field_io.cpp) ----------------------------------------
    def write_field_csv(self, grid, values, path):
        v = np.ascontiguousarray(values, dtype=np.float64)
        self._check(self.lib.orc_write_field_csv(C.byref(grid_struct(grid).c), _dp(v), str(path).encode()))

    def write_pgm(self, grid, values, path):
        v = np.ascontiguousarray(values, dtype=np.float64)
        self._check(self.lib.orc_write_pgm(C.byref(grid_struct(grid).c), _dp(v), str(path).encode()))

    def write_vtk(self, grid, arrays, path):
        """arrays: list of (name, values) in file order."""
        names = (C.c_char_p * len(arrays))(*[n.encode() for n, _ in arrays])
        vals = np.ascontiguousarray(np.concatenate([np.asarray(v, dtype=np.float64) for _, v in arrays]))
        self._check(self.lib.orc_write_vtk(C.byref(grid_struct(grid).c), len(arrays), names, _dp(vals),
                                           str(path).encode()))


_cache = {}


def load(which="port"):
    """Return the Oracle for "port" (C restatement) or "reference" (oracle/_ref)."""
    if which not in _cache:
        if which == "port":
            _cache[which] = Oracle(build_port())
        elif which == "reference":
            if not os.path.exists(REF_LIB):
                raise FileNotFoundError(REF_LIB)
            _cache[which] = Oracle(REF_LIB)
        else:
            raise ValueError(which)
    return _cache[which]


def has_reference():
    return os.path.exists(REF_LIB)


def ref_config_json(text):
    """Reference-only: parse_config + build_problem + build_schedule, as JSON."""
    import json

    lib = load("reference").lib
    lib.ref_config_json.restype = C.c_char_p
    return json.loads(lib.ref_config_json(text.encode()).decode())


def ref_check_config(text):
    """Reference-only: parse_config (+ validate_config); None or the ConfigError message."""
    lib = load("reference").lib
    lib.orc_last_error.restype = C.c_char_p
    rc = lib.ref_check_config(text.encode())
    return None if rc == 0 else lib.orc_last_error().decode()

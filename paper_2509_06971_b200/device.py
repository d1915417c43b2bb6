"""ctypes binding of include/petto_dev.h and a host-side mirror of the reference's
state-solver interface (StateOperator / StateHistory / hybrid_solve /
iterate_to_tolerance, /root/reference/proj/include/petto/state_solver.hpp).

The device library is mandatory: importing this module loads
lib/libpetto_b200.so and creating a context fails loudly without an sm_100 GPU.
There is no CPU fallback anywhere on this path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

MAX_PHASES = 8
OK, ABORT, INVALID, ERROR, IO = 0, 1, 2, 3, 4
MODE_FAST, MODE_REPLICA = 0, 1


class IoError(RuntimeError):
    """The reference's IoError (errors.hpp): a writer could not open or write a file."""


FIELD_STATE, FIELD_PHASE, FIELD_PROPERTY = 0, 1, 2


class PettoArray(C.Structure):
    _fields_ = [("field", C.c_int), ("index", C.c_int), ("name", C.c_char_p)]


class NumericalAbort(RuntimeError):
    """errors.hpp:10-23: carries the field name and the step index."""

    def __init__(self, message, step=None, field="state"):
        super().__init__(message)
        self.step = step
        self.field = field


class GridDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("n", C.c_int64 * 3), ("length", C.c_double * 3), ("physics", C.c_int),
        ("poisson_ratio", C.c_double), ("mode", C.c_int), ("device", C.c_int),
        ("k_begin", C.c_int64), ("k_end", C.c_int64), ("x_outermost", C.c_int),
    ]


class PTParams(C.Structure):
    _fields_ = [("dt_pt", C.c_double), ("dt_apt", C.c_double), ("theta", C.c_double), ("n_apt", C.c_long),
                ("n_pt", C.c_long), ("form", C.c_int)]


class SolveStats(C.Structure):
    _fields_ = [("iterations", C.c_long), ("r_initial", C.c_double), ("r_final", C.c_double),
                ("converged", C.c_int)]


class Material(C.Structure):
    _fields_ = [("kind", C.c_int), ("nphases", C.c_int), ("properties", C.c_double * MAX_PHASES),
                ("poisson_ratio", C.c_double), ("penalty", C.c_double), ("void_floor", C.c_double)]


class Targets(C.Structure):
    _fields_ = [("fractions", C.c_double * MAX_PHASES), ("has_region", C.c_int),
                ("region_fractions", C.c_double * MAX_PHASES), ("nregion", C.c_int64),
                ("region_nodes", C.POINTER(C.c_int64))]


class Weights(C.Structure):
    _fields_ = [("alpha_compliance", C.c_double), ("alpha_volume", C.c_double), ("alpha_unity", C.c_double),
                ("alpha_region", C.c_double), ("normalize_compliance", C.c_int), ("compliance_sign", C.c_int)]


class CHParams(C.Structure):
    _fields_ = [("mobility", C.c_double), ("gamma", C.c_double), ("dt", C.c_double)]


class CHStats(C.Structure):
    _fields_ = [("mass_before", C.c_double), ("mass_preclamp", C.c_double), ("mass_postclamp", C.c_double)]


class Report(C.Structure):
    _fields_ = [("compliance", C.c_double), ("volume", C.c_double), ("unity", C.c_double), ("region", C.c_double),
                ("volume_fractions", C.c_double * MAX_PHASES)]


class Schedule(C.Structure):
    _fields_ = [("pt", PTParams), ("ch", CHParams), ("max_loops", C.c_long), ("convergence_tol", C.c_double),
                ("convergence_window", C.c_int), ("report_every", C.c_int)]


class Record(C.Structure):
    _fields_ = [("loop", C.c_long), ("apt_steps", C.c_longlong), ("pt_steps", C.c_longlong),
                ("compliance", C.c_double), ("volume", C.c_double), ("unity", C.c_double), ("region", C.c_double),
                ("r_pde", C.c_double), ("separation", C.c_double), ("volume_fractions", C.c_double * MAX_PHASES),
                ("wall_seconds", C.c_double)]


class RunResult(C.Structure):
    _fields_ = [("loops", C.c_long), ("apt_steps", C.c_longlong), ("pt_steps", C.c_longlong),
                ("design_updates", C.c_longlong), ("ch_steps", C.c_longlong), ("clamp_mass_drift", C.c_double),
                ("termination", C.c_int), ("abort_detail", C.c_char * 256)]


RECORD_CB = C.CFUNCTYPE(None, C.POINTER(Record), C.c_void_p)

_lib = None


def lib():
    """Load (building if stale, when nvcc is present) the sm_100a library."""
    global _lib
    if _lib is None:
        path = os.environ.get("PETTO_B200_LIB") or _build.LIB  # A/B variants of the same C-ABI
        if path == _build.LIB and _build.stale():
            try:
                path = _build.build()
            except Exception:
                if not os.path.exists(path):
                    raise
        L = C.CDLL(path)
        L.petto_dev_version.restype = C.c_char_p
        L.petto_dev_last_error.restype = C.c_char_p
        L.petto_dev_last_error.argtypes = [C.c_void_p]
        L.petto_dev_stream.restype = C.c_void_p
        L.petto_dev_stream.argtypes = [C.c_void_p]
        L.petto_dev_spectral_bound.restype = C.c_double
        L.petto_dev_spectral_bound.argtypes = [C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_double,
                                               C.c_double]
        L.petto_dev_launch_count.restype = C.c_int64
        L.petto_dev_launch_count.argtypes = [C.c_void_p]
        for name in ("petto_dev_destroy",):
            getattr(L, name).argtypes = [C.c_void_p]
        _lib = L
    return _lib


EXPORTED = [
    "petto_dev_version", "petto_dev_device_count", "petto_dev_create", "petto_dev_destroy",
    "petto_dev_last_error", "petto_dev_stream", "petto_dev_set_mode", "petto_dev_set_constraints",
    "petto_dev_set_source", "petto_dev_set_property", "petto_dev_set_lame", "petto_dev_init_operator", "petto_dev_set_state",
    "petto_dev_get_state", "petto_dev_residual", "petto_dev_hybrid_solve", "petto_dev_iterate_to_tolerance",
    "petto_dev_set_design", "petto_dev_set_phases", "petto_dev_get_phases", "petto_dev_interpolate",
    "petto_dev_design_update", "petto_dev_ch_step", "petto_dev_objectives", "petto_dev_run",
    "petto_dev_unit_cell_stiffness", "petto_dev_spectral_bound", "petto_dev_launch_count",
    "petto_dev_kernel_timing", "petto_dev_kernel_stats", "petto_dev_comm_unique_id", "petto_dev_comm_init",
    "petto_dev_group_link", "petto_dev_group_hybrid_solve", "petto_dev_group_residual", "petto_dev_group_iterate_to_tolerance", "petto_dev_group_interpolate",
    "petto_dev_group_init_operator",
    "petto_dev_group_design_update", "petto_dev_group_ch_step", "petto_dev_group_objectives", "petto_dev_group_run",
    "petto_dev_peer_export", "petto_dev_peer_import",
    "petto_dev_write_field_csv", "petto_dev_write_vtk", "petto_dev_write_pgm", "petto_dev_format_values",
]


def comm_unique_id():
    """128-byte NCCL unique id (rank 0), to be broadcast by the caller."""
    buf = (C.c_ubyte * 128)()
    rc = lib().petto_dev_comm_unique_id(buf)
    if rc != OK:
        raise RuntimeError(lib().petto_dev_last_error(None).decode())
    return bytes(buf)


def group_link(ctxs):
    arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    ctxs[0]._check(lib().petto_dev_group_link(arr, len(ctxs)))


def _group(ctxs):
    return (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])


def group_hybrid_solve(ctxs, params):
    """hybrid_solve on a linked group of slab contexts (one process)."""
    step = C.c_int64(0)
    ctxs[0]._check(lib().petto_dev_group_hybrid_solve(_group(ctxs), len(ctxs), C.byref(pt_params(params)),
                                                      C.byref(step)))


def group_residual(ctxs):
    """residual_norm of the whole decomposed grid (the residual stays on the slabs)."""
    r = C.c_double(0.0)
    ctxs[0]._check(lib().petto_dev_group_residual(_group(ctxs), len(ctxs), C.byref(r)))
    return r.value


def group_iterate_to_tolerance(ctxs, mode, params, target, max_iters):
    st = SolveStats()
    ctxs[0]._check(lib().petto_dev_group_iterate_to_tolerance(_group(ctxs), len(ctxs), int(mode),
                                                              C.byref(pt_params(params)), C.c_double(target),
                                                              C.c_long(max_iters), C.byref(st)))
    return st


def group_interpolate(ctxs):
    ctxs[0]._check(lib().petto_dev_group_interpolate(_group(ctxs), len(ctxs)))


def group_init_operator(ctxs):
    ctxs[0]._check(lib().petto_dev_group_init_operator(_group(ctxs), len(ctxs)))


def group_design_update(ctxs):
    ctxs[0]._check(lib().petto_dev_group_design_update(_group(ctxs), len(ctxs)))


def group_ch_step(ctxs, mobility, gamma, dt):
    st = (CHStats * ctxs[0].nphases)()
    ctxs[0]._check(lib().petto_dev_group_ch_step(_group(ctxs), len(ctxs), C.byref(CHParams(mobility, gamma, dt)), st))
    return [(s.mass_before, s.mass_preclamp, s.mass_postclamp) for s in st]


def group_objectives(ctxs):
    rep = Report()
    sep = C.c_double(0.0)
    ctxs[0]._check(lib().petto_dev_group_objectives(_group(ctxs), len(ctxs), C.byref(rep), C.byref(sep)))
    return rep, sep.value


def group_run(ctxs, sched, callback=None):
    """run() (optimizer.hpp:120-223) over a linked group of slab contexts."""
    return ctxs[0]._run(sched, callback, lambda s, cb, res: lib().petto_dev_group_run(
        _group(ctxs), len(ctxs), C.byref(s), cb, None, C.byref(res)))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def unit_cell_stiffness(dim, h, nu):
    n = (1 << dim) * dim
    out = np.zeros(n * n)
    lib().petto_dev_unit_cell_stiffness(dim, (C.c_double * 3)(*h), C.c_double(nu), _dp(out))
    return out.reshape(n, n)


def spectral_bound(grid, nu, e_max):
    """elasticity_spectral_bound (state_solver.hpp:254-279) on the product's host code."""
    return lib().petto_dev_spectral_bound(grid.dim, (C.c_int64 * 3)(*grid.n), (C.c_double * 3)(*grid.length),
                                          C.c_double(nu), C.c_double(e_max))


def pt_params(p):
    return PTParams(p.dt_pt, p.dt_apt, p.theta, p.n_apt, p.n_pt, p.form)


class Context:
    """One problem resident in HBM (a petto_ctx)."""

    def __init__(self, grid, physics, poisson_ratio=0.3, mode=MODE_FAST, device=0, k_range=None,
                 x_outermost=False):
        """k_range: this slab's planes of the outermost device axis -- z, or x with
        x_outermost (the device keeps (y, z, x); uploads / downloads permute)."""
        L = lib()
        self.grid = grid
        self.physics = physics
        self.comps = grid.dim if physics else 1
        self.N = grid.num_nodes
        kb, ke = k_range if k_range else (0, 0)
        d = GridDesc(grid.dim, (C.c_int64 * 3)(*grid.n), (C.c_double * 3)(*grid.length), physics, poisson_ratio,
                     mode, device, kb, ke, 1 if x_outermost else 0)
        h = C.c_void_p()
        rc = L.petto_dev_create(C.byref(d), C.byref(h))
        if rc != OK:
            self._raise(rc, L.petto_dev_last_error(None).decode())
        self.h = h
        self._cb_keep = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().petto_dev_destroy(h)
            self.h = None

    close = __del__

    # -- errors: the reference's exception types ---------------------------
    def _raise(self, rc, msg=None):
        if msg is None:
            msg = lib().petto_dev_last_error(self.h).decode()
        if rc == ABORT:
            step = None
            if " at step " in msg:
                try:
                    step = int(msg.split(" at step ")[1].split(":")[0])
                except ValueError:
                    pass
            raise NumericalAbort(msg, step)
        if rc == INVALID:
            raise ValueError(msg)
        if rc == IO:
            raise IoError(msg)
        raise RuntimeError(msg)

    def _check(self, rc):
        if rc != OK:
            self._raise(rc)

    # -- uploads -------------------------------------------------------------
    def set_mode(self, mode):
        self._check(lib().petto_dev_set_mode(self.h, mode))

    def set_constraints(self, entries, values):
        e = np.ascontiguousarray(entries, dtype=np.int64)
        v = _f64(values)
        self._check(lib().petto_dev_set_constraints(self.h, e.ctypes.data_as(C.POINTER(C.c_int64)), _dp(v),
                                                    C.c_int64(len(e))))

    def set_source(self, source):
        self._check(lib().petto_dev_set_source(self.h, _dp(_f64(source))))

    def set_property(self, prop):
        self._check(lib().petto_dev_set_property(self.h, _dp(_f64(prop))))

    def set_lame(self, lam, mu):
        self._check(lib().petto_dev_set_lame(self.h, _dp(_f64(lam)), _dp(_f64(mu))))

    def init_operator(self):
        self._check(lib().petto_dev_init_operator(self.h))

    def set_state(self, cur, prev=None):
        c = _f64(cur)
        p = _f64(prev) if prev is not None else c
        self._check(lib().petto_dev_set_state(self.h, _dp(c), _dp(p)))

    def get_state(self, out_cur=None, out_prev=None):
        """Download the history; pass (pinned) arrays to avoid allocating."""
        c = out_cur if out_cur is not None else np.zeros(self.comps * self.N)
        p = out_prev if out_prev is not None else np.zeros(self.comps * self.N)
        assert c.dtype == np.float64 and c.flags.c_contiguous and p.dtype == np.float64 and p.flags.c_contiguous
        self._check(lib().petto_dev_get_state(self.h, _dp(c), _dp(p)))
        return c, p

    # -- state solve -----------------------------------------------------------
    def residual(self):
        out = np.zeros(self.comps * self.N)
        r = C.c_double(0.0)
        self._check(lib().petto_dev_residual(self.h, _dp(out), C.byref(r)))
        return out, r.value

    def hybrid_solve(self, params):
        step = C.c_int64(0)
        self._check(lib().petto_dev_hybrid_solve(self.h, C.byref(pt_params(params)), C.byref(step)))

    def iterate_to_tolerance(self, mode, params, target, max_iters):
        st = SolveStats()
        self._check(lib().petto_dev_iterate_to_tolerance(self.h, int(mode), C.byref(pt_params(params)),
                                                         C.c_double(target), C.c_long(max_iters), C.byref(st)))
        return st

    # -- design subsystems ----------------------------------------------------
    def set_design(self, kind, properties, poisson_ratio, penalty, void_floor, fractions, weights,
                   region_nodes=None, region_fractions=None):
        m = Material(kind, len(properties), (C.c_double * MAX_PHASES)(*properties), poisson_ratio, penalty,
                     void_floor)
        self._region = np.ascontiguousarray(region_nodes if region_nodes is not None else [0], dtype=np.int64)
        t = Targets((C.c_double * MAX_PHASES)(*fractions), 1 if region_fractions is not None else 0,
                    (C.c_double * MAX_PHASES)(*(region_fractions or [])),
                    len(region_nodes) if region_nodes is not None else 0,
                    self._region.ctypes.data_as(C.POINTER(C.c_int64)))
        w = Weights(weights.alpha_compliance, weights.alpha_volume, weights.alpha_unity, weights.alpha_region,
                    1 if weights.normalize_compliance else 0, int(weights.compliance_sign))
        self.nphases = len(properties)
        self._check(lib().petto_dev_set_design(self.h, C.byref(m), C.byref(t), C.byref(w)))

    def set_phases(self, phases):
        self._check(lib().petto_dev_set_phases(self.h, _dp(_f64(phases))))

    def get_phases(self, out=None):
        """Download the phases (a slab fills its owned planes of `out`)."""
        out = out if out is not None else np.zeros(self.nphases * self.N)
        self._check(lib().petto_dev_get_phases(self.h, _dp(out)))
        return out

    def interpolate(self, download=True):
        out = np.zeros(self.N) if download else None
        self._check(lib().petto_dev_interpolate(self.h, _dp(out) if download else None))
        return out

    def design_update(self):
        self._check(lib().petto_dev_design_update(self.h))

    def ch_step(self, mobility, gamma, dt):
        st = (CHStats * self.nphases)()
        self._check(lib().petto_dev_ch_step(self.h, C.byref(CHParams(mobility, gamma, dt)), st))
        return [(s.mass_before, s.mass_preclamp, s.mass_postclamp) for s in st]

    def objectives(self):
        rep = Report()
        sep = C.c_double(0.0)
        self._check(lib().petto_dev_objectives(self.h, C.byref(rep), C.byref(sep)))
        return rep, sep.value

    def run(self, sched, callback=None):
        """run() (optimizer.hpp:120-223); returns (RunResult, [Record])."""
        return self._run(sched, callback, lambda s, cb, res: lib().petto_dev_run(self.h, C.byref(s), cb, None,
                                                                                 C.byref(res)))

    def _run(self, sched, callback, call):
        s = Schedule(pt_params(sched.pt), CHParams(sched.ch_mobility, sched.ch_gamma, sched.dt_ch),
                     sched.max_loops, sched.convergence_tol, sched.convergence_window, sched.report_every)
        records = []

        def _cb(rec, _user):
            r = rec.contents
            copy = Record()
            C.pointer(copy)[0] = r
            records.append(copy)
            if callback:
                callback(copy)

        cb = RECORD_CB(_cb)
        res = RunResult()
        self._check(call(s, cb, res))
        return res, records

    @staticmethod
    def from_problem(prob, mode=MODE_FAST, device=0, k_range=None, x_outermost=False):
        """Upload a problem.Problem (build_problem's product) as run() expects it."""
        ctx = Context(prob.grid, prob.physics, prob.poisson_ratio, mode, device, k_range, x_outermost)
        ctx.set_constraints(prob.cons_entry, prob.cons_value)
        ctx.set_source(prob.source)
        ctx.set_design(prob.physics, prob.properties, prob.poisson_ratio, prob.penalty, prob.void_floor,
                       prob.fractions, prob.weights, prob.region_nodes if prob.has_region else None,
                       prob.region_fractions)
        ctx.set_phases(prob.initial_phases)
        ctx.set_state(prob.initial_state, prob.initial_state)
        return ctx

    def comm_init(self, uid, rank, nranks):
        """Join the NCCL communicator of the slab decomposition (one GPU per rank)."""
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        self._check(lib().petto_dev_comm_init(self.h, buf, int(rank), int(nranks)))

    PEER_BLOB_BYTES = 512

    def peer_export(self):
        """IPC handles of this slab's state buffers and step inbox (peer halo)."""
        buf = (C.c_ubyte * self.PEER_BLOB_BYTES)()
        self._check(lib().petto_dev_peer_export(self.h, buf))
        return bytes(buf)

    def peer_import(self, lo=None, hi=None):
        """Map the -1 / +1 neighbours' blobs (None at a physical end)."""
        lb = (C.c_ubyte * self.PEER_BLOB_BYTES).from_buffer_copy(lo) if lo else None
        hb = (C.c_ubyte * self.PEER_BLOB_BYTES).from_buffer_copy(hi) if hi else None
        self._check(lib().petto_dev_peer_import(self.h, lb, hb))

    # -- instrumentation -------------------------------------------------------
    # -- output writers (field_io.cpp) ---------------
    def write_field_csv(self, field, index, path):
        self._check(lib().petto_dev_write_field_csv(self.h, field, index, str(path).encode()))

    def write_vtk(self, arrays, path):
        """arrays: [(field, index, name), ...] in file order."""
        arr = (PettoArray * len(arrays))(*[PettoArray(f, i, n.encode()) for f, i, n in arrays])
        self._check(lib().petto_dev_write_vtk(self.h, arr, len(arrays), str(path).encode()))

    def write_pgm(self, field, index, path):
        self._check(lib().petto_dev_write_pgm(self.h, field, index, str(path).encode()))

    def format_values(self, values, sep_mode=0, row=1):
        """'%.17g' of every value (host array or device pointer), formatted on the device."""
        v = np.ascontiguousarray(values, dtype=np.float64)
        cap = 25 * len(v) + 1
        out = C.create_string_buffer(cap)
        n = C.c_int64()
        self._check(lib().petto_dev_format_values(self.h, v.ctypes.data_as(C.c_void_p), len(v), sep_mode,
                                                   max(1, row), out, cap, C.byref(n)))
        return out.raw[: n.value]

    def stream(self):
        return lib().petto_dev_stream(self.h)

    def launch_count(self):
        return lib().petto_dev_launch_count(self.h)

    def kernel_timing(self, enable=True, stride=1):
        """CUDA events around every `stride`-th hot launch (kernel_stats averages them)."""
        self._check(lib().petto_dev_kernel_timing(self.h, max(1, int(stride)) if enable else 0))

    def kernel_stats(self):
        ms, n, b = C.c_double(), C.c_int64(), C.c_double()
        name = C.create_string_buffer(64)
        self._check(lib().petto_dev_kernel_stats(self.h, C.byref(ms), C.byref(n), C.byref(b), name, 64))
        return ms.value, n.value, b.value, name.value.decode()


# ----------------------------------------------------------------------------
# Host-buffer mirror of the reference's operator interface.


@dataclass
class StateHistory:
    """StateHistory<double> (state_solver.hpp:37-45) on host arrays."""

    current: np.ndarray
    previous: np.ndarray

    @staticmethod
    def of(init):
        a = _f64(init)
        return StateHistory(a.copy(), a.copy())


class DeviceOperator:
    """A StateOperator (state_solver.hpp:65-72) whose residual runs on the B200."""

    def __init__(self, grid, physics, prop, source, bc, poisson_ratio=0.3, mode=MODE_FAST):
        from .problem import make_constraints

        self.grid = grid
        self.ctx = Context(grid, physics, poisson_ratio, mode)
        self._comps = self.ctx.comps
        self.cs = make_constraints(grid, bc, self._comps)
        self.ctx.set_constraints(*self.cs)
        self.ctx.set_source(source)
        self.ctx.set_property(prop)
        self.ctx.init_operator()

    def components(self):
        return self._comps

    def constraints(self):
        return self.cs

    def residual(self, state):
        self.ctx.set_state(state, state)
        return self.ctx.residual()[0]


def HeatOperator(grid, kappa, source, bc, mode=MODE_FAST):
    """HeatOperator (state_solver.hpp:76-95)."""
    return DeviceOperator(grid, 0, kappa, source, bc, mode=mode)


def ElasticityOperator(grid, modulus, nu, loads, bc, mode=MODE_FAST):
    """ElasticityOperator built from a Young's modulus field via make_lame (state_solver.hpp:289-325)."""
    return DeviceOperator(grid, 1, modulus, loads, bc, poisson_ratio=nu, mode=mode)


def residual_norm(r, nodes):
    """residual_norm (state_solver.hpp:49-58) -- host helper for host arrays."""
    r = _f64(r)
    return float(np.sqrt(np.dot(r, r)) / nodes)


def hybrid_solve(hist: StateHistory, op: DeviceOperator, params):
    """hybrid_solve (state_solver.hpp:480-498): uploads the history, runs on the
    device, downloads the new history (also on NumericalAbort)."""
    op.ctx.set_state(hist.current, hist.previous)
    try:
        op.ctx.hybrid_solve(params)
    finally:
        hist.current, hist.previous = op.ctx.get_state()


def iterate_to_tolerance(hist: StateHistory, op: DeviceOperator, mode, params, target, max_iters):
    """iterate_to_tolerance (state_solver.hpp:511-541)."""
    op.ctx.set_state(hist.current, hist.previous)
    try:
        return op.ctx.iterate_to_tolerance(mode, params, target, max_iters)
    finally:
        hist.current, hist.previous = op.ctx.get_state()

"""Python mirror of the reference gliosim API over the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference C++ library
(/root/reference/proj/include/gliosim/*.hpp) so the parity tests read like the
reference's own tests:

  reference (C++)                                this module
  ---------------------------------------------  --------------------------------------
  Grid (grid.hpp:14-51)                          Grid
  SimConfig (config.hpp:15-55)                   SimConfig
  classify / resample / diffusion_from_materials  classify / resample / diffusion_from_materials
    (imaging.hpp:35-41)
  assemble_diffusion (stencil.hpp:20)            assemble_diffusion -> StencilOperator
  SparseOperator::apply / one_norm (sparse.hpp)  StencilOperator.apply / one_norm
  select_params / expmv / phi1v (expact.hpp)     select_params / expmv / phi1v
  seed_initial / step / run (integrator.hpp)     seed_initial / step / run
  std::invalid_argument                          ValueError
  gliosim::numeric_error / data_error            NumericError / DataError

Every compute call goes to the GPU through the native library; nothing here computes
on the CPU beyond argument checks and the libm-parity seed (done in the library).
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


class NumericError(RuntimeError):
    """gliosim::numeric_error (errors.hpp:15-17)."""


class DataError(RuntimeError):
    """gliosim::data_error (errors.hpp:10-13)."""


class CudaError(RuntimeError):
    """Device / driver failure (no reference analogue)."""


def _raise(code: int, msg: str):
    if code == N.GS_EINVAL:
        raise ValueError(msg)
    if code == N.GS_ENUMERIC:
        raise NumericError(msg)
    if code == N.GS_EDATA:
        raise DataError(msg)
    raise CudaError(msg)


# ------------------------------------------------------------------------------------
# core types
# ------------------------------------------------------------------------------------

@dataclass
class Grid:
    """grid.hpp:14-51: lattice point (i,j,k) 1-based at origin + (i-1)h ..."""
    nx: int = 2
    ny: int = 2
    nz: int = 1
    h: float = 1.0
    origin: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1 or self.nz < 1:
            raise ValueError("Grid: point counts must be >= 1")
        if not self.h > 0.0:
            raise ValueError("Grid: spacing h must be positive")

    @property
    def shape(self):
        return (self.nx, self.ny, self.nz)

    def num_points(self) -> int:
        return self.nx * self.ny * self.nz

    def contains(self, p) -> bool:
        for a, n in enumerate(self.shape):
            lo = self.origin[a]
            hi = self.origin[a] + (n - 1) * self.h
            if p[a] < lo or p[a] > hi:
                return False
        return True


@dataclass
class SimConfig:
    """config.hpp:15-55 defaults (the 50^3 reference run)."""
    rho: float = 0.025
    d_white: float = 0.13
    d_gray: float = 0.013
    exp_tol: float = 1e-8
    nx: int = 50
    ny: int = 50
    nz: int = 50
    h: float = 200.0 / 49.0
    origin: tuple = (0.0, 0.0, 0.0)
    t0: float = 150.0
    t_end: float = 3500.0
    num_steps: int = 100
    seed_center: tuple = (102.0, 138.0, 96.0)
    seed_amplitude: float = 0.1
    seed_width: float = 10.0
    threshold_air: int = 1
    threshold_white: int = 230
    threshold_gray: int = 240
    threshold_max: int = 255
    slice_thickness: float = 1.0
    snapshot_every: int = 2
    front_threshold: float = 0.1

    def grid(self) -> Grid:
        return Grid(self.nx, self.ny, self.nz, self.h, tuple(self.origin))

    def tau(self) -> float:
        return (self.t_end - self.t0) / self.num_steps

    def validate(self):
        """config.cpp:53-77, same keys and messages."""
        def fail(key, why):
            raise DataError(f"config: key '{key}' {why}")
        if self.rho < 0.0: fail("rho", "must be >= 0")
        if self.d_gray < 0.0: fail("d_gray", "must be >= 0")
        if self.d_white < self.d_gray: fail("d_white", "must be >= d_gray")
        if not (0.0 < self.exp_tol < 1.0): fail("exp_tol", "must lie in (0,1)")
        if self.nx < 1: fail("nx", "must be >= 1")
        if self.ny < 1: fail("ny", "must be >= 1")
        if self.nz < 1: fail("nz", "must be >= 1")
        if not self.h > 0.0: fail("h", "must be positive")
        if not self.t_end > self.t0: fail("t_end", "must be greater than t0")
        if self.num_steps < 1: fail("num_steps", "must be >= 1")
        if not self.seed_amplitude >= 0.0: fail("amplitude", "must be >= 0")
        if not self.seed_width >= 0.0: fail("width", "must be >= 0")
        if self.threshold_air < 0: fail("threshold_air", "must be >= 0")
        if self.threshold_white <= self.threshold_air: fail("threshold_white", "must exceed threshold_air")
        if self.threshold_gray <= self.threshold_white: fail("threshold_gray", "must exceed threshold_white")
        if self.threshold_max < self.threshold_gray or self.threshold_max > 255:
            fail("threshold_max", "must lie in [threshold_gray, 255]")
        if self.slice_thickness < 0.0: fail("slice_thickness", "must be >= 0")
        if self.snapshot_every < 1: fail("snapshot_every", "must be >= 1")
        if not (0.0 < self.front_threshold < 1.0): fail("front_threshold", "must lie in (0,1)")


def time_at(cfg_or_tg, n: int) -> float:
    """TimeGrid::time (integrator.hpp:24-26): the last node is t_end exactly."""
    t0, t_end, steps = cfg_or_tg.t0, cfg_or_tg.t_end, cfg_or_tg.num_steps
    return t_end if n >= steps else t0 + n * ((t_end - t0) / steps)


@dataclass
class StepMetrics:
    """integrator.hpp:30-37."""
    step: int = 0
    time: float = 0.0
    total_mass: float = 0.0
    max_density: float = 0.0
    min_density: float = 0.0
    radius: float = 0.0


@dataclass
class RunTimings:
    assemble_seconds: float = 0.0
    step_seconds: float = 0.0
    io_seconds: float = 0.0


@dataclass
class RunResult:
    metrics: list = field(default_factory=list)
    u: np.ndarray | None = None
    timings: RunTimings = field(default_factory=RunTimings)
    infos: list = field(default_factory=list)  # per-step (s, m, terms) parity log


# ------------------------------------------------------------------------------------
# the operator (device resident)
# ------------------------------------------------------------------------------------

class StencilOperator:
    """The matrix-free device form of assemble_diffusion's SparseOperator.

    Owns one gs_ctx (device buffers + stream).  ``dim`` / ``one_norm`` / ``apply``
    mirror SparseOperator (sparse.hpp:13-38).
    """

    def __init__(self, grid: Grid, device: int = 0):
        self.lib = N.load()
        self.grid = grid
        h = C.c_void_p()
        rc = self.lib.gs_create(C.byref(h), grid.nx, grid.ny, grid.nz, float(grid.h), device)
        if rc != N.GS_OK:
            _raise(rc, self.lib.gs_last_error(None).decode("utf-8", "surrogateescape"))
        self.ctx = h

    # -- lifetime ----------------------------------------------------------------------
    def close(self):
        if getattr(self, "ctx", None):
            self.lib.gs_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc):
        if rc != N.GS_OK:
            _raise(rc, self.lib.gs_last_error(self.ctx).decode("utf-8", "surrogateescape"))

    # -- construction -------------------------------------------------------------------
    @classmethod
    def from_labels(cls, grid: Grid, labels, d_white=0.13, d_gray=0.013, device=0):
        op = cls(grid, device)
        op._check(op.lib.gs_set_labels(op.ctx, np.ascontiguousarray(labels, dtype=np.uint8).ravel(), d_white, d_gray))
        return op

    @classmethod
    def from_intensity(cls, grid: Grid, stack, width, height, slices, cfg: SimConfig | None = None, device=0):
        cfg = cfg or SimConfig()
        op = cls(grid, device)
        op._check(op.lib.gs_set_intensity(op.ctx, np.ascontiguousarray(stack, dtype=np.uint8).ravel(), width, height,
                                          slices, cfg.threshold_air, cfg.threshold_white, cfg.threshold_gray,
                                          cfg.d_white, cfg.d_gray))
        return op

    @classmethod
    def from_diffusion(cls, grid: Grid, d, device=0):
        op = cls(grid, device)
        op._check(op.lib.gs_set_diffusion(op.ctx, np.ascontiguousarray(d, dtype=np.float64).ravel()))
        return op

    # -- SparseOperator surface --------------------------------------------------------
    def dim(self) -> int:
        return self.grid.num_points()

    def one_norm(self) -> float:
        out = C.c_double()
        self._check(self.lib.gs_one_norm(self.ctx, C.byref(out)))
        return out.value

    def apply(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.size != self.dim():
            raise ValueError(f"SparseOperator::apply: vector length {x.size} != dim {self.dim()}")
        y = np.empty_like(x)
        self._check(self.lib.gs_apply(self.ctx, x, y))
        return y

    def labels(self) -> np.ndarray:
        out = np.empty(self.dim(), dtype=np.uint8)
        self._check(self.lib.gs_get_labels(self.ctx, out))
        return out

    def diffusion(self) -> np.ndarray:
        out = np.empty(self.dim(), dtype=np.float64)
        self._check(self.lib.gs_get_diffusion(self.ctx, out))
        return out

    # -- resident state ------------------------------------------------------------------
    def set_state(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        if u.size != self.dim():
            raise ValueError("run: initial state length does not match the grid")
        self._check(self.lib.gs_set_state(self.ctx, u))

    def get_state(self) -> np.ndarray:
        out = np.empty(self.dim(), dtype=np.float64)
        self._check(self.lib.gs_get_state(self.ctx, out))
        return out

    def state_device_ptr(self) -> int:
        return self.lib.gs_state_device_ptr(self.ctx)

    def stream_handle(self) -> int:
        return self.lib.gs_stream(self.ctx)

    def set_trace(self, capacity: int):
        """Record per-phase grid-barrier timestamps in later launches (diagnostics)."""
        self._check(self.lib.gs_set_trace(self.ctx, capacity))
        self._trace_cap = capacity

    def trace(self):
        """[(tag, ns)] of the last launch; see gliosim_b200.h for the tags."""
        cap = getattr(self, "_trace_cap", 0)
        buf = np.zeros(2 * max(cap, 1), dtype=np.uint64)
        n = C.c_int()
        self._check(self.lib.gs_get_trace(self.ctx, buf, cap, C.byref(n)))
        return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(n.value)]

    def uses_cluster(self) -> bool:
        """True when gs_run takes the small-grid single-cluster path."""
        return bool(self.lib.gs_uses_cluster(self.ctx))

    def uses_flat2d(self) -> bool:
        """True when the Taylor loop takes the resident-tile 2-D path (cluster-path runs aside)."""
        return bool(self.lib.gs_uses_flat2d(self.ctx))

    def set_kernel_timing(self, enable: bool):
        """CUDA-event timing of every kernel launch of later calls (on the context's stream)."""
        self._check(self.lib.gs_set_kernel_timing(self.ctx, 1 if enable else 0))

    def kernel_times(self):
        """{kernel: (total ms, launches)} of the last call: prep, border, taylor, update."""
        ms = np.zeros(4, dtype=np.float64)
        n = np.zeros(4, dtype=np.int32)
        self._check(self.lib.gs_get_kernel_times(self.ctx, ms, n))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(["prep", "border", "taylor", "update"])}

    def snapshot_vtk(self, path, labels=None):
        """Queue the resident state as a VTK snapshot (gs_snapshot_vtk): device copy now,
        host copy on a side stream, formatting on a writer thread.  Errors of earlier
        snapshots surface here or in flush_snapshots()."""
        lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.uint8).ravel()
        if lab is not None and lab.size != self.dim():
            raise ValueError("write_vtk: material volume does not match the field grid")
        self._check(self.lib.gs_snapshot_vtk(self.ctx, os.fsencode(path), N.d3(self.grid.origin),
                                             lab.ctypes.data if lab is not None else None))

    def flush_snapshots(self):
        self._check(self.lib.gs_snapshot_flush(self.ctx))

    def step_resident(self, rho, tau, tol, info=True):
        inf = N.GsStepInfo() if info else None
        self._check(self.lib.gs_step(self.ctx, rho, tau, tol, C.byref(inf) if inf is not None else None))
        return inf

    def run_resident(self, n_steps, rho, tau, tol, origin=(0.0, 0.0, 0.0), center=(0.0, 0.0, 0.0),
                     front_threshold=0.1, metrics=True, infos=False):
        """The time loop on the resident state: one device launch for n_steps steps."""
        m = (N.GsMetrics * (n_steps + 1))() if metrics else None
        inf = (N.GsStepInfo * max(1, n_steps))() if infos else None
        self._check(self.lib.gs_run(self.ctx, n_steps, rho, tau, tol, N.d3(origin), N.d3(center), front_threshold,
                                    C.cast(m, C.c_void_p) if m is not None else None,
                                    C.cast(inf, C.c_void_p) if inf is not None else None))
        return m, inf


class CsrOperator(StencilOperator):
    """A generic SparseOperator (sparse.hpp:13-38) on the GPU: CSR with sorted, unique columns,
    validated like the reference's constructor (sparse.cpp:14-35)."""

    def __init__(self, offs, cols, vals, device: int = 0):
        self.lib = N.load()
        offs = np.ascontiguousarray(offs, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int32)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        n = len(offs) - 1
        self.grid = Grid(max(n, 1), 1, 1, 1.0)
        h = C.c_void_p()
        rc = self.lib.gs_create_csr(C.byref(h), n, offs, cols, vals, device)
        if rc != N.GS_OK:
            _raise(rc, self.lib.gs_last_error(None).decode("utf-8", "surrogateescape"))
        self.ctx = h


# ------------------------------------------------------------------------------------
# free functions with the reference's names
# ------------------------------------------------------------------------------------

def classify(intensity: int, cfg: SimConfig | None = None) -> int:
    """imaging.cpp:118-123 (scalar convenience; volumes go through resample on the GPU)."""
    cfg = cfg or SimConfig()
    if intensity <= cfg.threshold_air:
        return 0
    if intensity <= cfg.threshold_white:
        return 1
    if intensity <= cfg.threshold_gray:
        return 2
    return 3


def resample(stack, width: int, height: int, slices: int, grid: Grid, cfg: SimConfig | None = None) -> np.ndarray:
    """imaging.cpp:125-141 on the GPU (K1); returns the MaterialVolume labels."""
    if slices < 1 or width < 1 or height < 1:
        raise DataError("resample: degenerate stack")
    with StencilOperator.from_intensity(grid, stack, width, height, slices, cfg) as op:
        return op.labels()


def diffusion_from_materials(labels, cfg: SimConfig | None = None) -> np.ndarray:
    """imaging.cpp:143-153 as a host table lookup (the device keeps labels + table)."""
    cfg = cfg or SimConfig()
    table = np.array([0.0, cfg.d_white, cfg.d_gray, 0.0])
    return table[np.asarray(labels, dtype=np.uint8)]


def assemble_diffusion(grid: Grid, d) -> StencilOperator:
    """stencil.cpp:5-43: the device keeps the operator matrix-free."""
    return StencilOperator.from_diffusion(grid, d)


def select_params(norm_tA: float, tol: float):
    lib = N.load()
    s, m = C.c_int(), C.c_int()
    rc = lib.gs_select_params(norm_tA, tol, C.byref(s), C.byref(m))
    if rc != N.GS_OK:
        _raise(rc, lib.gs_last_error(None).decode("utf-8", "surrogateescape"))
    return s.value, m.value


def _vec(a: StencilOperator, b, who):
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.size != a.dim():
        raise ValueError(f"{who}: vector length does not match operator dimension")
    return b


def expmv(t: float, a: StencilOperator, b, tol: float, info: bool = False):
    b = _vec(a, b, "expmv")
    out = np.empty_like(b)
    inf = N.GsStepInfo()
    a._check(a.lib.gs_expmv(a.ctx, t, b, tol, out, C.byref(inf)))
    return (out, inf) if info else out


def phi1v(t: float, a: StencilOperator, b, tol: float, info: bool = False):
    b = _vec(a, b, "phi1v")
    out = np.empty_like(b)
    inf = N.GsStepInfo()
    a._check(a.lib.gs_phi1v(a.ctx, t, b, tol, out, C.byref(inf)))
    return (out, inf) if info else out


def step(a: StencilOperator, u, rho: float, tau: float, tol: float, info: bool = False):
    """integrator.cpp:52-63 with value semantics: the step runs on a staging buffer, so the
    operator's resident state (run_resident / set_state) is left untouched.  A length mismatch
    raises what the reference's first use of u raises, SparseOperator::apply's message
    (sparse.cpp:44-46 via integrator.cpp:55)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    if u.size != a.dim():
        raise ValueError(f"SparseOperator::apply: vector length {u.size} != dim {a.dim()}")
    out = np.empty_like(u)
    inf = N.GsStepInfo()
    a._check(a.lib.gs_step_host(a.ctx, u, rho, tau, tol, out, C.byref(inf)))
    return (out, inf) if info else out


def seed_initial(a: StencilOperator, cfg: SimConfig, mask: bool = True) -> np.ndarray:
    """integrator.cpp:32-50 (host libm, bit-identical to the reference); lattice points are
    placed by the operator's grid (grid.point, grid.hpp:35-37), as seed_initial(d, cfg) does."""
    u = np.empty(a.dim(), dtype=np.float64)
    a._check(a.lib.gs_seed_initial(a.ctx, N.d3(a.grid.origin), cfg.seed_amplitude, cfg.seed_width,
                                   N.d3(cfg.seed_center), 1 if mask else 0, u))
    return u


def run_ensemble(ops, n_steps: int, rhos, tau: float, tol: float, origins=None, centers=None,
                 front_threshold: float = 0.1, metrics: bool = True, infos: bool = False, groups: int = 0):
    """gs_run_ensemble: every member (a StencilOperator with its resident state) advances
    n_steps steps of run()'s loop (integrator.cpp:91-138), batched over the members.
    Returns (metrics, infos): per member a list of GsMetrics nodes / GsStepInfo records (or
    None)."""
    ops = list(ops)
    n = len(ops)
    if n == 0:
        raise ValueError("run_ensemble: no members")
    lib = ops[0].lib
    rhos = np.ascontiguousarray(rhos, dtype=np.float64)
    if rhos.size != n:
        raise ValueError("run_ensemble: one rho per member")
    org = np.ascontiguousarray(origins if origins is not None else np.zeros((n, 3)), dtype=np.float64).reshape(n, 3)
    cen = np.ascontiguousarray(centers if centers is not None else np.zeros((n, 3)), dtype=np.float64).reshape(n, 3)
    ctxs = (C.c_void_p * n)(*[o.ctx for o in ops])
    m = (N.GsMetrics * (n * (n_steps + 1)))() if metrics else None
    inf = (N.GsStepInfo * max(1, n * n_steps))() if infos else None
    rc = lib.gs_run_ensemble(ctxs, n, n_steps, rhos, tau, tol, org.ctypes.data_as(C.c_void_p),
                             cen.ctypes.data_as(C.c_void_p), front_threshold,
                             C.cast(m, C.c_void_p) if m is not None else None,
                             C.cast(inf, C.c_void_p) if inf is not None else None, groups)
    if rc != N.GS_OK:
        _raise(rc, lib.gs_last_error(ops[0].ctx).decode("utf-8", "surrogateescape"))
    per_m = [list(m[i * (n_steps + 1):(i + 1) * (n_steps + 1)]) for i in range(n)] if m is not None else None
    per_i = [list(inf[i * n_steps:(i + 1) * n_steps]) for i in range(n)] if inf is not None else None
    return per_m, per_i


def step_ensemble_host(ops, us, rhos, tau: float, tol: float, outs=None, infos: bool = False, groups: int = 0,
                       chunks: int = 0):
    """gs_step_ensemble_host: one exponential-Euler step of every member with host vectors
    (step() per member, integrator.cpp:52-63), batched, the copies overlapping the other member
    chunks' steps.  `us` / `outs`: one float64 vector per member (pinned memory makes the
    copies asynchronous).  Returns (outs, infos or None)."""
    ops = list(ops)
    n = len(ops)
    if n == 0:
        raise ValueError("run_ensemble: no members")
    lib = ops[0].lib
    rhos = np.ascontiguousarray(rhos, dtype=np.float64)
    if rhos.size != n or len(us) != n:
        raise ValueError("run_ensemble: one rho and one state per member")
    ins = [np.ascontiguousarray(u, dtype=np.float64) for u in us]
    for op, u in zip(ops, ins):
        if u.size != op.grid.num_points():
            raise ValueError("step: state length does not match the grid")
    if outs is None:
        outs = [np.empty_like(u) for u in ins]
    else:
        outs = list(outs)
        if len(outs) != n:
            raise ValueError("step_ensemble: one output vector per member")
        for op, o in zip(ops, outs):
            # the library writes n doubles through each pointer: exact dtype, size and layout
            if (not isinstance(o, np.ndarray) or o.dtype != np.float64 or not o.flags.c_contiguous
                    or not o.flags.writeable or o.size != op.grid.num_points()):
                raise ValueError("step_ensemble: each output must be a writeable C-contiguous float64 array "
                                 "with one value per grid point")
    pin = (C.c_void_p * n)(*[u.ctypes.data for u in ins])
    pout = (C.c_void_p * n)(*[o.ctypes.data for o in outs])
    ctxs = (C.c_void_p * n)(*[o.ctx for o in ops])
    inf = (N.GsStepInfo * n)() if infos else None
    rc = lib.gs_step_ensemble_host(ctxs, n, pin, pout, rhos, tau, tol,
                                   C.cast(inf, C.c_void_p) if inf is not None else None, groups, chunks)
    if rc != N.GS_OK:
        _raise(rc, lib.gs_last_error(ops[0].ctx).decode("utf-8", "surrogateescape"))
    return outs, (list(inf) if inf is not None else None)


def run(cfg: SimConfig, a: StencilOperator, u0, snapshot=None, on_range=None, on_step=None,
        with_infos: bool = False, _vtk=None) -> RunResult:
    """integrator.cpp:91-138: the time loop runs on the GPU as one launch sequence per segment
    between snapshots (per step when a StepWatcher or RangeWarning is given, so they fire
    live); metrics are computed on the device at every node, then the hooks fire in order
    with the reference's arguments.

    _vtk = (out_dir, labels or None) is run_to_directory's sink (pipeline.cpp:39-45):
    snapshot_NNNN.vtk files written asynchronously by the native library."""
    cfg.validate()
    grid = a.grid
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    if u0.size != grid.num_points():
        raise ValueError("run: initial state length does not match the grid")
    res = RunResult()
    a.set_state(u0)
    tau = cfg.tau()
    sinks = snapshot is not None or _vtk is not None
    # segment ends: snapshot nodes (0, every snapshot_every, the last; integrator.cpp:112,
    # :135-136); with a StepWatcher / RangeWarning every step, so the hooks fire live, after
    # each step as in the reference's loop (integrator.cpp:128-131) -- a failing step then
    # leaves the hooks of every completed step fired
    if on_step or on_range:
        cuts = list(range(1, cfg.num_steps + 1))
    elif sinks:
        cuts = [n for n in range(1, cfg.num_steps + 1) if n % cfg.snapshot_every == 0 or n == cfg.num_steps]
    else:
        cuts = [cfg.num_steps]

    def emit(n):
        tic = time.perf_counter()
        if snapshot:
            snapshot(n, time_at(cfg, n), a.get_state())
        if _vtk is not None:
            a.snapshot_vtk(os.path.join(_vtk[0], "snapshot_%04d.vtk" % n), _vtk[1])
        res.timings.io_seconds += time.perf_counter() - tic

    emit(0)
    done = 0
    all_metrics = []
    for cut in cuts:
        k = cut - done
        tic = time.perf_counter()
        # metrics on the operator's grid (compute_metrics uses grid.point of the DiffusionField's
        # grid, integrator.cpp:65-89), as seeding and the snapshots do
        m, inf = a.run_resident(k, cfg.rho, tau, cfg.exp_tol, grid.origin, cfg.seed_center, cfg.front_threshold,
                                metrics=True, infos=with_infos)
        res.timings.step_seconds += time.perf_counter() - tic
        first = 0 if done == 0 else 1
        for q in range(first, k + 1):
            node = done + q
            sm = StepMetrics(node, time_at(cfg, node), m[q].total_mass, m[q].max_density, m[q].min_density,
                             m[q].radius)
            all_metrics.append(sm)
            if node == 0:
                continue
            # hooks in the reference's order (integrator.cpp:128-131)
            if on_step:
                on_step(sm)
            if on_range and (sm.min_density < -0.01 or sm.max_density > 1.01):
                on_range(sm.step, sm.min_density, sm.max_density)
        if with_infos:
            res.infos.extend(inf[q].as_dict() for q in range(k))
        done = cut
        if sinks and (cut % cfg.snapshot_every == 0 or cut == cfg.num_steps):
            emit(cut)
    if _vtk is not None:
        tic = time.perf_counter()
        a._check(a.lib.gs_snapshot_flush(a.ctx))
        res.timings.io_seconds += time.perf_counter() - tic
    res.metrics = all_metrics
    res.u = a.get_state()
    return res


# file formats and run_to_directory (vtk.cpp, imaging.cpp, pipeline.cpp)
from .fileio import (DiffusionField, ImageStack, MaterialVolume, ScalarField, load_raw_volume,  # noqa: E402,F401
                     load_stack, matter_fractions, read_label_volume, read_vtk, run_to_directory,
                     stencil_from_stack, uniform_diffusion, uniform_labels, write_label_volume,
                     write_metrics_csv, write_vtk)

"""ctypes bindings for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two checkers live here:

* ``Port``  -- ``oracle/liboracle.so``, our plain-C restatement of the reference hot
  path (``gliosim_oracle.c``; each function cites the reference file:line).
* ``Ref``   -- ``oracle/_ref/libgliosim_ref.so``, the UNMODIFIED reference library
  compiled from /root/reference/proj/src by ``oracle/Makefile`` plus our extern "C"
  wrapper ``ref_capi.cpp``.  Present only where it was built (it travels to the GPU
  box as an untracked build artefact); tests that need it skip otherwise.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference
arm may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgliosim_ref.so")
REF_SRC = "/root/reference/proj"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

MAX_STAGES = 256


class OrOp(C.Structure):
    pass


OrOp._fields_ = [
    ("kind", C.c_int),
    ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
    ("h", C.c_double),
    ("d", C.c_void_p),
    ("dim", C.c_int64),
    ("offs", C.c_void_p), ("cols", C.c_void_p), ("vals", C.c_void_p),
    ("base", C.c_void_p), ("border", C.c_void_p), ("b", C.c_void_p),
]


class OrLog(C.Structure):
    _fields_ = [
        ("s", C.c_int), ("m", C.c_int), ("branch", C.c_int),
        ("total_terms", C.c_int64),
        ("terms", C.c_int * MAX_STAGES),
        ("bnorm", C.c_double), ("anorm", C.c_double), ("coln", C.c_double),
        ("gamma", C.c_double), ("norm_tA", C.c_double),
    ]

    def stage_terms(self):
        return [self.terms[i] for i in range(min(self.s, MAX_STAGES))]


def build_port():
    """Compile the C restatement if missing (gcc is in the image, here and on the box)."""
    if not os.path.exists(PORT_SO):
        subprocess.check_call(["make", "-s", "-C", HERE, "liboracle.so"])
    return PORT_SO


def build_ref():
    """Compile the reference where its sources exist (build container only)."""
    if os.path.isdir(REF_SRC) and not os.path.exists(REF_SO):
        subprocess.check_call(["make", "-s", "-j8", "-C", HERE, "ref"])
    return REF_SO if os.path.exists(REF_SO) else None


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"oracle error {code}: {what}")
        self.code = code


class Port:
    """The C restatement."""

    def __init__(self):
        self.lib = C.CDLL(build_port())
        L = self.lib
        L.or_classify.argtypes = [C.c_int] * 4
        L.or_nearest_source.argtypes = [C.c_int] * 3
        L.or_resample.argtypes = [_u8p] + [C.c_int] * 9 + [_u8p]
        L.or_resample.restype = None
        L.or_diffusion_from_labels.argtypes = [_u8p, C.c_int64, C.c_double, C.c_double, _dp]
        L.or_diffusion_from_labels.restype = None
        L.or_op_apply.argtypes = [C.POINTER(OrOp), _dp, _dp]
        L.or_op_apply.restype = None
        L.or_op_one_norm.argtypes = [C.POINTER(OrOp)]
        L.or_op_one_norm.restype = C.c_double
        L.or_stencil_colsums.argtypes = [C.POINTER(OrOp), _dp]
        L.or_stencil_colsums.restype = None
        L.or_select_params.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.or_expmv.argtypes = [C.c_double, C.POINTER(OrOp), _dp, C.c_double, _dp, C.POINTER(OrLog)]
        L.or_phi1v_ex.argtypes = [C.c_double, C.POINTER(OrOp), _dp, C.c_double, _dp, C.POINTER(OrLog),
                                  C.c_void_p, C.c_void_p]
        L.or_step_ex.argtypes = [C.POINTER(OrOp), _dp, C.c_double, C.c_double, C.c_double, _dp,
                                 C.POINTER(OrLog), C.c_void_p, C.c_void_p]
        L.or_seed_initial.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _dp, C.c_double, C.c_double,
                                      _dp, C.c_void_p, _dp]
        L.or_seed_initial.restype = None
        L.or_compute_metrics.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double, _dp, _dp, C.c_double, _dp]
        L.or_compute_metrics.restype = None
        L.or_run.argtypes = [C.POINTER(OrOp), _dp, C.c_int, C.c_double, C.c_double, C.c_double, _dp, _dp,
                             C.c_double, _dp, C.c_void_p]

    # -- operators ------------------------------------------------------------------
    @staticmethod
    def stencil(shape, h, d):
        """shape = (nx, ny, nz); d float64 x-fastest.  Keeps d alive on the op."""
        d = np.ascontiguousarray(d, dtype=np.float64).ravel()
        op = OrOp()
        op.kind = 0
        op.nx, op.ny, op.nz = (int(s) for s in shape)
        op.h = float(h)
        op.d = d.ctypes.data
        op._keep = (d,)
        return op

    @staticmethod
    def csr(offs, cols, vals):
        offs = np.ascontiguousarray(offs, dtype=np.int64)
        cols = np.ascontiguousarray(cols, dtype=np.int32)
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        op = OrOp()
        op.kind = 1
        op.dim = len(offs) - 1
        op.offs, op.cols, op.vals = offs.ctypes.data, cols.ctypes.data, vals.ctypes.data
        op._keep = (offs, cols, vals)
        return op

    @staticmethod
    def dim(op):
        return op.nx * op.ny * op.nz if op.kind == 0 else op.dim

    def apply(self, op, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.dim(op), dtype=np.float64)
        self.lib.or_op_apply(C.byref(op), x, y)
        return y

    def one_norm(self, op):
        return self.lib.or_op_one_norm(C.byref(op))

    def colsums(self, op):
        y = np.empty(self.dim(op), dtype=np.float64)
        self.lib.or_stencil_colsums(C.byref(op), y)
        return y

    # -- exponential action ---------------------------------------------------------
    def select_params(self, norm, tol):
        s, m = C.c_int(), C.c_int()
        rc = self.lib.or_select_params(norm, tol, C.byref(s), C.byref(m))
        if rc:
            raise OracleError(rc, "select_params")
        return s.value, m.value

    def expmv(self, t, op, b, tol):
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty_like(b)
        log = OrLog()
        rc = self.lib.or_expmv(t, C.byref(op), b, tol, out, C.byref(log))
        if rc:
            raise OracleError(rc, "expmv")
        return out, log

    def phi1v(self, t, op, b, tol, bnorm=None, coln=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty_like(b)
        log = OrLog()
        bn = C.c_double(bnorm) if bnorm is not None else None
        cn = C.c_double(coln) if coln is not None else None
        rc = self.lib.or_phi1v_ex(t, C.byref(op), b, tol, out, C.byref(log),
                                  C.cast(C.byref(bn), C.c_void_p) if bn is not None else None,
                                  C.cast(C.byref(cn), C.c_void_p) if cn is not None else None)
        if rc:
            raise OracleError(rc, "phi1v")
        return out, log

    def step(self, op, u, rho, tau, tol, bnorm=None, coln=None):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty_like(u)
        log = OrLog()
        bn = C.c_double(bnorm) if bnorm is not None else None
        cn = C.c_double(coln) if coln is not None else None
        rc = self.lib.or_step_ex(C.byref(op), u, rho, tau, tol, out, C.byref(log),
                                 C.cast(C.byref(bn), C.c_void_p) if bn is not None else None,
                                 C.cast(C.byref(cn), C.c_void_p) if cn is not None else None)
        if rc:
            raise OracleError(rc, "step")
        return out, log

    def seed_initial(self, shape, h, amplitude, width, center, d_mask=None, origin=(0.0, 0.0, 0.0)):
        nx, ny, nz = shape
        u = np.empty(nx * ny * nz, dtype=np.float64)
        dm = None if d_mask is None else np.ascontiguousarray(d_mask, dtype=np.float64)
        self.lib.or_seed_initial(nx, ny, nz, h, np.array(origin, dtype=np.float64), amplitude, width,
                                 np.array(center, dtype=np.float64),
                                 None if dm is None else dm.ctypes.data, u)
        return u

    def compute_metrics(self, u, shape, h, center, front_threshold=0.1, origin=(0.0, 0.0, 0.0)):
        out = np.empty(4, dtype=np.float64)
        self.lib.or_compute_metrics(np.ascontiguousarray(u, dtype=np.float64), *shape, h,
                                    np.array(origin, dtype=np.float64), np.array(center, dtype=np.float64),
                                    front_threshold, out)
        return out

    def run(self, op, u0, n_steps, rho, tau, tol, center, front_threshold=0.1, origin=(0.0, 0.0, 0.0),
            with_logs=False):
        u = np.array(u0, dtype=np.float64, copy=True)
        metrics = np.empty((n_steps + 1) * 4, dtype=np.float64)
        logs = (OrLog * n_steps)() if with_logs else None
        rc = self.lib.or_run(C.byref(op), u, n_steps, rho, tau, tol, np.array(origin, dtype=np.float64),
                             np.array(center, dtype=np.float64), front_threshold, metrics,
                             C.cast(logs, C.c_void_p) if logs is not None else None)
        if rc:
            raise OracleError(rc, "run")
        return u, metrics.reshape(n_steps + 1, 4), (list(logs) if logs is not None else None)

    # -- material map ---------------------------------------------------------------
    def classify(self, v, t_air=1, t_white=230, t_gray=240):
        return self.lib.or_classify(v, t_air, t_white, t_gray)

    def nearest_source(self, i, n, src):
        return self.lib.or_nearest_source(i, n, src)

    def resample(self, stack, w, hgt, slices, shape, t_air=1, t_white=230, t_gray=240):
        labels = np.empty(shape[0] * shape[1] * shape[2], dtype=np.uint8)
        self.lib.or_resample(np.ascontiguousarray(stack, dtype=np.uint8).ravel(), w, hgt, slices,
                             *shape, t_air, t_white, t_gray, labels)
        return labels

    def diffusion_from_labels(self, labels, d_white=0.13, d_gray=0.013):
        labels = np.ascontiguousarray(labels, dtype=np.uint8).ravel()
        d = np.empty(labels.size, dtype=np.float64)
        self.lib.or_diffusion_from_labels(labels, labels.size, d_white, d_gray, d)
        return d


class Ref:
    """The unmodified reference library (via ref_capi.cpp)."""

    def __init__(self, path=None):
        path = path or build_ref()
        if not path or not os.path.exists(path):
            raise FileNotFoundError("reference library not built (oracle/_ref missing)")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_stencil_step.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _dp, _dp, C.c_double,
                                       C.c_double, C.c_double, C.c_int, _dp]
        L.ref_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _dp, _dp, C.c_int, C.c_double,
                              C.c_double, C.c_double, C.c_double, _dp, C.c_double, C.c_int,
                              C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
        L.ref_stencil_apply.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _dp, _dp, _dp]
        L.ref_stencil_one_norm.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _dp, C.POINTER(C.c_double)]
        L.ref_resample.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _u8p]
        L.ref_diffusion_from_labels.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _dp]
        L.ref_seed_initial.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _dp,
                                       C.c_void_p, _dp]
        L.ref_classify.argtypes = [C.c_int]
        L.ref_select_params.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_int)]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode("utf-8", "surrogateescape"))

    def step(self, shape, h, d, u, rho, tau, tol, workers=1):
        out = np.empty(len(u), dtype=np.float64)
        self._check(self.lib.ref_stencil_step(*shape, h, np.ascontiguousarray(d, dtype=np.float64),
                                              np.ascontiguousarray(u, dtype=np.float64), rho, tau, tol,
                                              workers, out))
        return out

    def run(self, shape, h, d, u0, n_steps, rho, t0, t_end, tol, center, front_threshold=0.1, workers=1):
        n = shape[0] * shape[1] * shape[2]
        u = np.empty(n, dtype=np.float64)
        metrics = np.empty((n_steps + 1) * 4, dtype=np.float64)
        secs = C.c_double()
        self._check(self.lib.ref_run(*shape, h, np.ascontiguousarray(d, dtype=np.float64),
                                     np.ascontiguousarray(u0, dtype=np.float64), n_steps, rho, t0, t_end, tol,
                                     np.array(center, dtype=np.float64), front_threshold, workers,
                                     u.ctypes.data, metrics.ctypes.data, C.byref(secs)))
        return u, metrics.reshape(n_steps + 1, 4), secs.value

    def apply(self, shape, h, d, x):
        y = np.empty(len(x), dtype=np.float64)
        self._check(self.lib.ref_stencil_apply(*shape, h, np.ascontiguousarray(d, dtype=np.float64),
                                               np.ascontiguousarray(x, dtype=np.float64), y))
        return y

    def one_norm(self, shape, h, d):
        out = C.c_double()
        self._check(self.lib.ref_stencil_one_norm(*shape, h, np.ascontiguousarray(d, dtype=np.float64),
                                                  C.byref(out)))
        return out.value

    def resample(self, stack, w, hgt, slices, shape):
        labels = np.empty(shape[0] * shape[1] * shape[2], dtype=np.uint8)
        self._check(self.lib.ref_resample(np.ascontiguousarray(stack, dtype=np.uint8).ravel(), w, hgt, slices,
                                          *shape, labels))
        return labels

    def diffusion_from_labels(self, labels, shape):
        d = np.empty(shape[0] * shape[1] * shape[2], dtype=np.float64)
        self._check(self.lib.ref_diffusion_from_labels(np.ascontiguousarray(labels, dtype=np.uint8), *shape, d))
        return d

    def seed_initial(self, shape, h, amplitude, width, center, d_mask=None):
        u = np.empty(shape[0] * shape[1] * shape[2], dtype=np.float64)
        dm = None if d_mask is None else np.ascontiguousarray(d_mask, dtype=np.float64)
        self._check(self.lib.ref_seed_initial(*shape, h, amplitude, width, np.array(center, dtype=np.float64),
                                              None if dm is None else dm.ctypes.data, u))
        return u

    def classify(self, v):
        return self.lib.ref_classify(v)

    # ---- file formats (vtk.cpp, imaging.cpp, pipeline.cpp) ------------------------------
    def _files(self):
        L = self.lib
        if getattr(self, "_files_typed", False):
            return L
        cp, vp, ip = C.c_char_p, C.c_void_p, C.POINTER(C.c_int)
        L.ref_write_vtk.argtypes = [cp, _dp, C.c_int, C.c_int, C.c_int, C.c_double, _dp, vp]
        L.ref_read_vtk.argtypes = [cp, ip, C.POINTER(C.c_double), _dp, vp, C.c_int64]
        L.ref_write_metrics_csv.argtypes = [cp, C.c_int, vp, vp, vp]
        L.ref_load_stack.argtypes = [C.POINTER(cp), C.c_int, ip, vp, C.c_int64]
        L.ref_load_raw_volume.argtypes = [cp, ip, vp, C.c_int64]
        L.ref_write_label_volume.argtypes = [cp, _u8p, C.c_int, C.c_int, C.c_int]
        L.ref_read_label_volume.argtypes = [cp, C.c_int, C.c_int, C.c_int, _u8p]
        L.ref_matter_fractions.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double)]
        L.ref_run_to_directory.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _dp, vp, C.c_int, C.c_int,
                                           C.c_double, C.c_double, C.c_double, C.c_double, _dp, C.c_double,
                                           C.c_double, cp, vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        self._files_typed = True
        return L

    def write_vtk(self, path, u, shape, h, origin=(0.0, 0.0, 0.0), labels=None):
        lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.uint8)
        self._check(self._files().ref_write_vtk(os.fsencode(path), np.ascontiguousarray(u, dtype=np.float64),
                                                *shape, h, np.array(origin, dtype=np.float64),
                                                None if lab is None else lab.ctypes.data))

    def read_vtk(self, path):
        """-> (dims, h, origin, values)"""
        L = self._files()
        dims = (C.c_int * 3)()
        h = C.c_double()
        origin = np.zeros(3)
        self._check(L.ref_read_vtk(os.fsencode(path), dims, C.byref(h), origin, None, 0))
        vals = np.empty(dims[0] * dims[1] * dims[2])
        self._check(L.ref_read_vtk(os.fsencode(path), dims, C.byref(h), origin, vals.ctypes.data, vals.size))
        return tuple(dims), h.value, tuple(origin), vals

    def write_metrics_csv(self, path, steps, times, m4):
        st = np.ascontiguousarray(steps, dtype=np.int32)
        tm = np.ascontiguousarray(times, dtype=np.float64)
        mm = np.ascontiguousarray(m4, dtype=np.float64).reshape(-1, 4)
        n = len(st)
        self._check(self._files().ref_write_metrics_csv(os.fsencode(path), n, st.ctypes.data if n else None,
                                                        tm.ctypes.data if n else None,
                                                        mm.ctypes.data if n else None))

    def load_stack(self, paths):
        L = self._files()
        arr = (C.c_char_p * max(1, len(paths)))(*[os.fsencode(p) for p in paths])
        dims = (C.c_int * 3)()
        self._check(L.ref_load_stack(arr, len(paths), dims, None, 0))
        out = np.empty(dims[0] * dims[1] * dims[2], dtype=np.uint8)
        self._check(L.ref_load_stack(arr, len(paths), dims, out.ctypes.data, out.size))
        return tuple(dims), out

    def load_raw_volume(self, path):
        L = self._files()
        dims = (C.c_int * 3)()
        self._check(L.ref_load_raw_volume(os.fsencode(path), dims, None, 0))
        out = np.empty(dims[0] * dims[1] * dims[2], dtype=np.uint8)
        self._check(L.ref_load_raw_volume(os.fsencode(path), dims, out.ctypes.data, out.size))
        return tuple(dims), out

    def write_label_volume(self, path, labels, shape):
        self._check(self._files().ref_write_label_volume(os.fsencode(path),
                                                         np.ascontiguousarray(labels, dtype=np.uint8), *shape))

    def read_label_volume(self, path, shape):
        out = np.empty(shape[0] * shape[1] * shape[2], dtype=np.uint8)
        self._check(self._files().ref_read_label_volume(os.fsencode(path), *shape, out))
        return out

    def matter_fractions(self, labels, shape):
        w, g = C.c_double(), C.c_double()
        self._check(self._files().ref_matter_fractions(np.ascontiguousarray(labels, dtype=np.uint8), *shape,
                                                       C.byref(w), C.byref(g)))
        return w.value, g.value

    def run_to_directory(self, shape, h, d, labels, n_steps, snapshot_every, rho, t0, t_end, tol, center,
                         amplitude, width, out_dir):
        n = shape[0] * shape[1] * shape[2]
        u = np.empty(n)
        ss, io = C.c_double(), C.c_double()
        lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.uint8)
        self._check(self._files().ref_run_to_directory(
            *shape, h, np.ascontiguousarray(d, dtype=np.float64), None if lab is None else lab.ctypes.data,
            n_steps, snapshot_every, rho, t0, t_end, tol, np.array(center, dtype=np.float64), amplitude, width,
            os.fsencode(out_dir), u.ctypes.data, C.byref(ss), C.byref(io)))
        return u, ss.value, io.value

    def select_params(self, norm, tol):
        s, m = C.c_int(), C.c_int()
        self._check(self.lib.ref_select_params(norm, tol, C.byref(s), C.byref(m)))
        return s.value, m.value


def read_records(path):
    """Parse gen_golden's record stream into {name: ndarray}."""
    out = {}
    kinds = {0: (np.float64, 8), 1: (np.int64, 8), 2: (np.int32, 4)}
    with open(path, "rb") as f:
        data = f.read()
    pos = 0
    while pos < len(data):
        (ln,) = np.frombuffer(data, np.uint32, 1, pos)
        pos += 4
        name = data[pos:pos + ln].decode()
        pos += ln
        kind = data[pos]
        pos += 1
        (count,) = np.frombuffer(data, np.uint64, 1, pos)
        pos += 8
        dt, sz = kinds[kind]
        out[name] = np.frombuffer(data, dt, int(count), pos).copy()
        pos += int(count) * sz
    return out

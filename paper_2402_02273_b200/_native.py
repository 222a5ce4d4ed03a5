"""ctypes binding of the C-ABI (include/gliosim_b200.h).

The native library is the product: if it is missing this module raises -- there is
no Python or CPU fallback.  It is built in-tree by ``paper_2402_02273_b200.build``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libgliosim_b200.so")
MAX_STAGES = 256

GS_OK, GS_EINVAL, GS_ENUMERIC, GS_EDATA, GS_ECUDA = range(5)


class GsStepInfo(C.Structure):
    _fields_ = [
        ("s", C.c_int32), ("m", C.c_int32), ("branch", C.c_int32), ("reruns", C.c_int32),
        ("total_terms", C.c_int64),
        ("terms", C.c_int32 * MAX_STAGES),
        ("bnorm", C.c_double), ("anorm", C.c_double), ("coln", C.c_double),
        ("gamma", C.c_double), ("norm_tA", C.c_double),
    ]

    def stage_terms(self):
        return [self.terms[i] for i in range(min(self.s, MAX_STAGES))]

    def as_dict(self):
        return {"s": self.s, "m": self.m, "branch": self.branch, "total_terms": self.total_terms, "reruns": self.reruns,
                "terms": self.stage_terms(), "bnorm": self.bnorm, "anorm": self.anorm, "coln": self.coln,
                "gamma": self.gamma, "norm_tA": self.norm_tA}


class GsMetrics(C.Structure):
    _fields_ = [("total_mass", C.c_double), ("max_density", C.c_double), ("min_density", C.c_double),
                ("radius", C.c_double)]


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_d3 = C.POINTER(C.c_double)

_lib = None

EXPORTS = [
    "gs_create", "gs_create_csr", "gs_destroy", "gs_last_error", "gs_num_points", "gs_stream",
    "gs_set_intensity", "gs_set_labels", "gs_set_diffusion", "gs_get_labels", "gs_get_diffusion",
    "gs_one_norm", "gs_apply", "gs_set_state", "gs_get_state", "gs_state_device_ptr",
    "gs_select_params", "gs_expmv", "gs_phi1v", "gs_step", "gs_step_host", "gs_run", "gs_run_ensemble",
    "gs_step_ensemble_host",
    "gs_seed_initial",
    "gs_set_trace", "gs_get_trace", "gs_set_kernel_timing", "gs_get_kernel_times",
    "gs_write_vtk", "gs_read_vtk", "gs_write_metrics_csv", "gs_snapshot_vtk", "gs_snapshot_flush",
    "gs_load_stack", "gs_load_raw_volume", "gs_write_label_volume", "gs_read_label_volume",
    "gs_matter_fractions", "gs_uses_cluster", "gs_uses_flat2d",
]


def load(path: str | None = None):
    """Load (and type) the native library; raises if it is not built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"native library missing: {path} (build it: python -m paper_2402_02273_b200.build)")
    L = C.CDLL(path)
    vp = C.c_void_p
    L.gs_create.argtypes = [C.POINTER(vp), C.c_int, C.c_int, C.c_int, C.c_double, C.c_int]
    L.gs_create_csr.argtypes = [C.POINTER(vp), C.c_int64,
                                np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS"),
                                np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS"), _dp, C.c_int]
    L.gs_destroy.argtypes = [vp]
    L.gs_destroy.restype = None
    L.gs_last_error.argtypes = [vp]
    L.gs_last_error.restype = C.c_char_p
    L.gs_num_points.argtypes = [vp]
    L.gs_num_points.restype = C.c_int64
    L.gs_stream.argtypes = [vp]
    L.gs_stream.restype = vp
    L.gs_set_intensity.argtypes = [vp, _u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_double, C.c_double]
    L.gs_set_labels.argtypes = [vp, _u8p, C.c_double, C.c_double]
    L.gs_set_diffusion.argtypes = [vp, _dp]
    L.gs_get_labels.argtypes = [vp, _u8p]
    L.gs_get_diffusion.argtypes = [vp, _dp]
    L.gs_one_norm.argtypes = [vp, C.POINTER(C.c_double)]
    L.gs_apply.argtypes = [vp, _dp, _dp]
    L.gs_set_state.argtypes = [vp, _dp]
    L.gs_get_state.argtypes = [vp, _dp]
    L.gs_state_device_ptr.argtypes = [vp]
    L.gs_state_device_ptr.restype = vp
    L.gs_select_params.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.gs_expmv.argtypes = [vp, C.c_double, _dp, C.c_double, _dp, C.POINTER(GsStepInfo)]
    L.gs_phi1v.argtypes = [vp, C.c_double, _dp, C.c_double, _dp, C.POINTER(GsStepInfo)]
    L.gs_step.argtypes = [vp, C.c_double, C.c_double, C.c_double, C.POINTER(GsStepInfo)]
    L.gs_step_host.argtypes = [vp, _dp, C.c_double, C.c_double, C.c_double, _dp, C.POINTER(GsStepInfo)]
    L.gs_run.argtypes = [vp, C.c_int, C.c_double, C.c_double, C.c_double, _d3, _d3, C.c_double, vp, vp]
    L.gs_seed_initial.argtypes = [vp, _d3, C.c_double, C.c_double, _d3, C.c_int, _dp]
    if hasattr(L, "gs_run_ensemble"):
        L.gs_run_ensemble.argtypes = [C.POINTER(vp), C.c_int, C.c_int, _dp, C.c_double, C.c_double, vp, vp,
                                      C.c_double, vp, vp, C.c_int]
    if hasattr(L, "gs_step_ensemble_host"):
        L.gs_step_ensemble_host.argtypes = [C.POINTER(vp), C.c_int, C.POINTER(vp), C.POINTER(vp), _dp, C.c_double,
                                            C.c_double, vp, C.c_int, C.c_int]
    if hasattr(L, "gs_set_trace"):  # diagnostics
        L.gs_set_trace.argtypes = [vp, C.c_int]
        L.gs_get_trace.argtypes = [vp, np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS"), C.c_int,
                                   C.POINTER(C.c_int)]
    if hasattr(L, "gs_set_kernel_timing"):
        L.gs_set_kernel_timing.argtypes = [vp, C.c_int]
        L.gs_get_kernel_times.argtypes = [vp, np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS"),
                                          np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")]
    if hasattr(L, "gs_write_vtk"):  # file formats (vtk.cpp, imaging.cpp)
        cp, ip, i64 = C.c_char_p, C.POINTER(C.c_int), C.c_int64
        L.gs_write_vtk.argtypes = [cp, _dp, C.c_int, C.c_int, C.c_int, C.c_double, _d3, vp, C.c_int]
        L.gs_read_vtk.argtypes = [cp, ip, _d3, _d3, vp, i64, C.c_int]
        L.gs_write_metrics_csv.argtypes = [cp, C.c_int, vp, vp, vp]
        L.gs_snapshot_vtk.argtypes = [vp, cp, _d3, vp]
        L.gs_snapshot_flush.argtypes = [vp]
        L.gs_load_stack.argtypes = [C.POINTER(cp), C.c_int, ip, ip, ip, vp, i64]
        L.gs_load_raw_volume.argtypes = [cp, ip, ip, ip, vp, i64]
        L.gs_write_label_volume.argtypes = [cp, _u8p, C.c_int, C.c_int, C.c_int]
        L.gs_read_label_volume.argtypes = [cp, C.c_int, C.c_int, C.c_int, _u8p]
        L.gs_matter_fractions.argtypes = [vp, _d3, _d3]
    if hasattr(L, "gs_uses_cluster"):
        L.gs_uses_cluster.argtypes = [vp]
    if hasattr(L, "gs_uses_flat2d"):
        L.gs_uses_flat2d.argtypes = [vp]
    for name in EXPORTS:
        if name not in ("gs_destroy", "gs_last_error", "gs_num_points", "gs_stream", "gs_state_device_ptr") \
                and hasattr(L, name):
            getattr(L, name).restype = C.c_int
    if path == LIB_PATH:
        _lib = L
    return L


def d3(v):
    return (C.c_double * 3)(*[float(x) for x in v])

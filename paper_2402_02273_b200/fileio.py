"""File formats of the reference, backed by the native library (csrc/gs_io.cpp).

Mirrors (paths relative to /root/reference/proj):

  reference                                             here
  ----------------------------------------------------  -----------------------------------
  write_vtk(u, path, materials)  vtk.hpp:40-41          write_vtk(field, path, materials=None)
  read_vtk(path)                 vtk.hpp:44             read_vtk(path) -> ScalarField
  write_metrics_csv(series, p)   vtk.hpp:48             write_metrics_csv(series, path)
  load_stack(paths)              imaging.hpp:29         load_stack(paths) -> ImageStack
  load_raw_volume(path)          imaging.hpp:33         load_raw_volume(path) -> ImageStack
  write/read_label_volume        imaging.hpp:53-54      write_label_volume / read_label_volume
  matter_fractions(mv)           imaging.hpp:49         matter_fractions(op | MaterialVolume)
  uniform_diffusion / uniform_labels  pipeline.hpp:15-16
  run_to_directory               pipeline.hpp:18-24     run_to_directory(cfg, a, materials, out_dir, ...)

Output bytes are identical to the reference's (17 significant digits, vtk.cpp:16-20);
messages and exception types follow it (data_error -> DataError, invalid_argument ->
ValueError).
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import gliosim as G


def _free_check(lib, rc):
    if rc != N.GS_OK:
        G._raise(rc, lib.gs_last_error(None).decode("utf-8", "surrogateescape"))


def _path(p) -> bytes:
    return os.fsencode(p)


@dataclass
class ScalarField:
    """fields.hpp ScalarField: a grid and one value per lattice point (x fastest)."""
    grid: G.Grid
    values: np.ndarray


@dataclass
class ImageStack:
    """imaging.hpp:15-26: 8-bit slices, bottom first; pixel (x,y,z) at x + y*w + z*w*h."""
    width: int
    height: int
    num_slices: int
    intensities: np.ndarray

    def at(self, x: int, y: int, z: int) -> int:
        return int(self.intensities[x + y * self.width + z * self.width * self.height])


@dataclass
class MaterialVolume:
    """fields.hpp MaterialVolume: one Material code (0 Air, 1 White, 2 Gray, 3 Skull) per point."""
    grid: G.Grid
    labels: np.ndarray


@dataclass
class DiffusionField:
    """fields.hpp DiffusionField: one diffusion coefficient per point."""
    grid: G.Grid
    d: np.ndarray


def _labels_of(materials, n):
    if materials is None:
        return None
    lab = materials.labels if hasattr(materials, "labels") else materials
    lab = np.ascontiguousarray(lab, dtype=np.uint8).ravel()
    if lab.size != n:
        raise ValueError("write_vtk: material volume does not match the field grid")
    return lab


def write_vtk(u: ScalarField, path, materials=None, threads: int = 0):
    lib = N.load()
    g = u.grid
    vals = np.ascontiguousarray(u.values, dtype=np.float64).ravel()
    if vals.size != g.num_points():
        raise ValueError("write_vtk: field length does not match its grid")
    lab = _labels_of(materials, vals.size)
    _free_check(lib, lib.gs_write_vtk(_path(path), vals, g.nx, g.ny, g.nz, float(g.h), N.d3(g.origin),
                                      lab.ctypes.data if lab is not None else None, threads))


def read_vtk(path, threads: int = 0) -> ScalarField:
    lib = N.load()
    dims = (C.c_int * 3)()
    h = C.c_double()
    origin = (C.c_double * 3)()
    _free_check(lib, lib.gs_read_vtk(_path(path), dims, C.byref(h), origin, None, 0, threads))
    n = dims[0] * dims[1] * dims[2]
    vals = np.empty(n, dtype=np.float64)
    _free_check(lib, lib.gs_read_vtk(_path(path), dims, C.byref(h), origin, vals.ctypes.data, n, threads))
    return ScalarField(G.Grid(dims[0], dims[1], dims[2], h.value, tuple(origin)), vals)


def write_metrics_csv(series, path):
    lib = N.load()
    n = len(series)
    step = np.array([m.step for m in series], dtype=np.int32)
    tm = np.array([m.time for m in series], dtype=np.float64)
    met = np.array([[m.total_mass, m.max_density, m.min_density, m.radius] for m in series],
                   dtype=np.float64).reshape(n, 4)
    _free_check(lib, lib.gs_write_metrics_csv(_path(path), n, step.ctypes.data if n else None,
                                              tm.ctypes.data if n else None, met.ctypes.data if n else None))


def load_stack(paths) -> ImageStack:
    lib = N.load()
    paths = [os.fspath(p) for p in paths]
    arr = (C.c_char_p * max(1, len(paths)))(*[_path(p) for p in paths])
    w, h, s = C.c_int(), C.c_int(), C.c_int()
    _free_check(lib, lib.gs_load_stack(arr, len(paths), C.byref(w), C.byref(h), C.byref(s), None, 0))
    out = np.empty(w.value * h.value * s.value, dtype=np.uint8)
    _free_check(lib, lib.gs_load_stack(arr, len(paths), C.byref(w), C.byref(h), C.byref(s), out.ctypes.data,
                                       out.size))
    return ImageStack(w.value, h.value, s.value, out)


def load_raw_volume(path) -> ImageStack:
    lib = N.load()
    w, h, s = C.c_int(), C.c_int(), C.c_int()
    _free_check(lib, lib.gs_load_raw_volume(_path(path), C.byref(w), C.byref(h), C.byref(s), None, 0))
    out = np.empty(w.value * h.value * s.value, dtype=np.uint8)
    _free_check(lib, lib.gs_load_raw_volume(_path(path), C.byref(w), C.byref(h), C.byref(s), out.ctypes.data,
                                            out.size))
    return ImageStack(w.value, h.value, s.value, out)


def write_label_volume(mv: MaterialVolume, path):
    lib = N.load()
    g = mv.grid
    lab = np.ascontiguousarray(mv.labels, dtype=np.uint8).ravel()
    if lab.size != g.num_points():
        raise ValueError("write_label_volume: labels do not match the grid")
    _free_check(lib, lib.gs_write_label_volume(_path(path), lab, g.nx, g.ny, g.nz))


def read_label_volume(path, grid: G.Grid) -> MaterialVolume:
    lib = N.load()
    lab = np.empty(grid.num_points(), dtype=np.uint8)
    _free_check(lib, lib.gs_read_label_volume(_path(path), grid.nx, grid.ny, grid.nz, lab))
    return MaterialVolume(grid, lab)


def uniform_diffusion(grid: G.Grid, d: float) -> DiffusionField:
    """pipeline.cpp:16-21."""
    return DiffusionField(grid, np.full(grid.num_points(), float(d)))


def uniform_labels(grid: G.Grid, m: int) -> MaterialVolume:
    """pipeline.cpp:23-28."""
    return MaterialVolume(grid, np.full(grid.num_points(), int(m), dtype=np.uint8))


def matter_fractions(src):
    """imaging.cpp:155-164 on the device: (white, gray) shares of the tissue voxels.
    `src` is a StencilOperator built from labels, or a MaterialVolume (uploaded)."""
    if isinstance(src, G.StencilOperator):
        w, g = C.c_double(), C.c_double()
        src._check(src.lib.gs_matter_fractions(src.ctx, C.byref(w), C.byref(g)))
        return w.value, g.value
    with G.StencilOperator.from_labels(src.grid, src.labels) as op:
        return matter_fractions(op)


def stencil_from_stack(stack: ImageStack, grid: G.Grid, cfg: G.SimConfig | None = None, device: int = 0):
    """load_stack/load_raw_volume -> resample -> classify -> diffusion_from_materials on the GPU
    (imaging.cpp:118-153): the operator a run needs, straight from the loaded intensities."""
    return G.StencilOperator.from_intensity(grid, stack.intensities, stack.width, stack.height, stack.num_slices,
                                            cfg, device=device)


def run_to_directory(cfg: G.SimConfig, a, materials, out_dir, workers: int = 1, on_step=None,
                     on_range=None) -> G.RunResult:
    """pipeline.cpp:30-53: seed from cfg, run, write snapshot_NNNN.vtk at every snapshot node
    (with the material array when `materials` is given) and metrics.csv.

    Snapshots go through gs_snapshot_vtk: a device copy of the state, a side-stream copy to
    pinned memory and formatting on host threads while the GPU runs the next segment.
    `a` is a StencilOperator or a DiffusionField(grid, d)."""
    try:
        os.makedirs(out_dir, exist_ok=True)
    except OSError as e:
        raise G.DataError(f"cannot create output directory {out_dir}: {e}") from None
    own = not isinstance(a, G.StencilOperator)
    op = G.assemble_diffusion(a.grid, a.d) if own else a
    try:
        lab = _labels_of(materials, op.grid.num_points())
        u0 = G.seed_initial(op, cfg)
        res = G.run(cfg, op, u0, on_range=on_range, on_step=on_step, _vtk=(os.fspath(out_dir), lab))
        tic = time.perf_counter()
        write_metrics_csv(res.metrics, os.path.join(out_dir, "metrics.csv"))
        res.timings.io_seconds += time.perf_counter() - tic
        return res
    finally:
        if own:
            op.close()

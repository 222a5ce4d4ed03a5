"""BASELINE.json configurations C1..C5 as concrete, seeded workloads.

Shared by bench.py and the tests so the GPU path and the CPU oracle see identical
bytes.  Physical constants are the reference defaults (config.hpp:17-31): rho 0.025/day,
D_white 0.13, D_gray 0.013 mm^2/day, tol 1e-8, t0 150 d, tau 33.5 d; spacing
h = 200/(n-1) mm (the presets' 200 mm box, config.cpp:207, :215); Gaussian seed of
amplitude 1 and width 1/(2 (sigma h)^2) at a seeded interior white-matter voxel.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import phantom

RHO = 0.025
TAU = 33.5
T0 = 150.0
TOL = 1e-8
D_WHITE = 0.13
D_GRAY = 0.013
# classify thresholds (config.hpp:40-43)
T_AIR, T_WHITE, T_GRAY = 1, 230, 240


@dataclass(frozen=True)
class Workload:
    name: str
    nx: int
    ny: int
    nz: int
    steps: int
    sigma_vox: float
    seed: int
    perturb: float = 0.0
    seeds: int = 1            # Gaussian seed points
    stack_slices: int = 0     # > 0: build from a sparse axial stack resampled in z
    members: int = 1          # ensemble members
    rho_scale: float = 1.0
    note: str = ""

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def h(self) -> float:
        return 200.0 / (max(self.nx, self.ny, self.nz) - 1)

    @property
    def tau(self) -> float:
        return TAU

    @property
    def rho(self) -> float:
        return RHO * self.rho_scale

    @property
    def t_end(self) -> float:
        return T0 + self.steps * TAU


CONFIGS = [
    Workload("C1", 32, 32, 32, 100, 3.0, 101, note="3-D 32^3 fp64, 100 steps (reference default run size)"),
    Workload("C2", 256, 256, 1, 200, 4.0, 202, note="2-D 256^2 mid-plane slice, 200 steps"),
    Workload("C3", 128, 128, 128, 100, 3.0, 303, seeds=2, stack_slices=29,
             note="128^3 from a 29-slice 128x128 stack, NN-upsampled in z; two seeds"),
    Workload("C4", 256, 256, 256, 100, 6.0, 404, perturb=0.10,
             note="256^3 headline; shell radii perturbed +-10%; rho default (C4x4: 4x rho)"),
    Workload("C5", 128, 128, 128, 50, 3.0, 505, members=64,
             note="ensemble of 64 independent 128^3 runs, rho log-uniform in [0.25x, 4x]"),
]


def get(name: str) -> Workload:
    for w in CONFIGS:
        if w.name == name:
            return w
    if name == "C4x4":
        base = get("C4")
        return Workload("C4x4", base.nx, base.ny, base.nz, base.steps, base.sigma_vox, base.seed, base.perturb,
                        rho_scale=4.0, note="256^3 at 4x rho")
    raise KeyError(name)


def intensity(w: Workload, member: int = 0):
    """uint8 input volume (or stack) for the workload.

    Returns (data, width, height, slices): either the full nx*ny*nz volume or, for
    C3, the sparse 29-slice stack that the material map resamples in z."""
    seed = w.seed + 1000 * member
    if w.stack_slices:
        st = phantom.slice_stack(w.nx, w.ny, w.stack_slices, w.nz, seed)
        return st.ravel(), w.nx, w.ny, w.stack_slices
    if w.nz == 1:
        depth = max(w.nx, w.ny)
        v = phantom.shell_phantom(w.nx, w.ny, depth, seed, w.perturb, z_plane=depth // 2)
        return v.ravel(), w.nx, w.ny, 1
    v = phantom.shell_phantom(w.nx, w.ny, w.nz, seed, w.perturb)
    return v.ravel(), w.nx, w.ny, w.nz


def classify_table() -> np.ndarray:
    v = np.arange(256)
    return np.where(v <= T_AIR, 0, np.where(v <= T_WHITE, 1, np.where(v <= T_GRAY, 2, 3))).astype(np.uint8)


def seed_points(w: Workload, labels: np.ndarray, member: int = 0):
    """Seed centres in mm (0-based voxel * h) for the workload's Gaussian seeds."""
    out = []
    for s in range(w.seeds):
        i, j, k = phantom.pick_seed_voxel(labels, (w.nx, w.ny, w.nz), w.seed + 1000 * member, salt=5 + 7 * s,
                                          margin=1)
        out.append((i * w.h, j * w.h, k * w.h))
    return out


def seed_width(w: Workload) -> float:
    return 1.0 / (2.0 * (w.sigma_vox * w.h) ** 2)


def member_rho(w: Workload, member: int) -> float:
    """C5: rho log-uniform over [0.25, 4] x default (seeded)."""
    if w.members == 1:
        return w.rho
    u = float(phantom.uniform01(w.seed, 900 + member, 1)[0])
    return RHO * float(np.exp(np.log(0.25) + u * (np.log(4.0) - np.log(0.25))))

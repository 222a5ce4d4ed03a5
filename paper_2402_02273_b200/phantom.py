"""Seeded synthetic head phantoms (host-side workload generator).

The paper's 29-slice MRI stack is private and absent, so BASELINE.json's
configs are driven by synthetic uint8 intensity volumes with the same role: nested
ellipsoid shells -- from outside in air, skin, skull, gray matter, white matter -- each
with an intensity band plus uniform integer noise in [-10, +10] (clamped to [0, 255]).
Band centres are chosen against the reference classify thresholds
(config.hpp:40-43: Air <= 1 < White <= 230 < Gray <= 240 < Skull):

  air    0    no noise (noise on 0 would turn ~43% of air into percolating white
              matter)
  skin   252  -> Skull (the reference has no skin material; D = 0)
  skull  250  -> Skull, ~1/21 speckled into Gray
  gray   235  -> Gray 10/21, White 6/21, Skull 5/21 (partial-volume speckle)
  white  150  -> White

Noise comes from a counter-based generator (splitmix64 of seed and voxel index) so
the bytes are identical on every machine and independent of any libstdc++
distribution.  The same bytes feed the oracle and the CUDA path.

This module only generates inputs; it is not on the hot path.
"""
from __future__ import annotations

import numpy as np

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)

AIR, SKIN, SKULL, GRAY, WHITE = 0, 252, 250, 235, 150
# shell boundaries in normalised ellipsoidal radius (outer edge of each shell)
R_SKIN, R_SKULL, R_GRAY, R_WHITE = 1.00, 0.94, 0.86, 0.74
HEAD_AXES = (0.92, 0.80, 0.88)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & MASK64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & MASK64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & MASK64
        return z ^ (z >> np.uint64(31))


def _stream(seed: int, salt: int, count: int) -> np.ndarray:
    base = np.uint64((seed * 0x100000001B3 + salt * 0x9E37) & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        idx = np.arange(count, dtype=np.uint64) + (base << np.uint64(20))
    return splitmix64(idx)


def uniform01(seed: int, salt: int, count: int) -> np.ndarray:
    """Deterministic uniforms in [0, 1) from the counter-based stream."""
    return (_stream(seed, salt, count) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _perturbation(seed: int, amplitude: float):
    """Smooth seeded radial perturbation p(dir) with |p| <= amplitude."""
    if amplitude == 0.0:
        return None
    r = uniform01(seed, 77, 6 * 5)
    coef = r[0:6] + 0.25
    coef = coef / coef.sum() * amplitude
    freq = (r[6:24].reshape(6, 3) - 0.5) * 4.0  # |f| up to ~3.5 cycles per unit direction
    phase = r[24:30] * 2.0 * np.pi
    return coef, freq, phase


def shell_intensity(X, Y, Z, seed: int, vox_index: np.ndarray, perturb: float = 0.0) -> np.ndarray:
    """Intensity (uint8) at normalised coordinates X, Y, Z in [-1, 1] (box-relative)."""
    ax, ay, az = HEAD_AXES
    xe, ye, ze = X / ax, Y / ay, Z / az
    rho = np.sqrt(xe * xe + ye * ye + ze * ze)
    pert = _perturbation(seed, perturb)
    if pert is not None:
        coef, freq, phase = pert
        inv = 1.0 / np.maximum(rho, 1e-12)
        dx, dy, dz = xe * inv, ye * inv, ze * inv
        p = np.zeros_like(rho)
        for q in range(6):
            p += coef[q] * np.sin(2.0 * np.pi * (freq[q, 0] * dx + freq[q, 1] * dy + freq[q, 2] * dz) + phase[q])
        rho = rho / (1.0 + p)
    base = np.full(rho.shape, AIR, dtype=np.int32)
    base[rho <= R_SKIN] = SKIN
    base[rho <= R_SKULL] = SKULL
    base[rho <= R_GRAY] = GRAY
    base[rho <= R_WHITE] = WHITE
    with np.errstate(over="ignore"):
        z = splitmix64(vox_index.astype(np.uint64) + np.uint64((seed & 0xFFFFFFFF) << 32))
    nz = (z % np.uint64(21)).astype(np.int32) - 10
    val = np.where(base == AIR, 0, np.clip(base + nz, 0, 255))
    return val.astype(np.uint8)


def shell_phantom(nx: int, ny: int, nz: int, seed: int, perturb: float = 0.0, z_plane: int | None = None) -> np.ndarray:
    """x-fastest uint8 intensity volume of shape (nz, ny, nx).

    ``z_plane`` evaluates a single mid-plane slice of an ``nz``-deep volume (C2's
    2-D configuration); the result then has shape (1, ny, nx) and keeps the voxel
    indices (and hence noise) of that plane.
    """
    def axis(n):
        return np.zeros(1) if n == 1 else np.linspace(-1.0, 1.0, n)

    zs = np.arange(nz) if z_plane is None else np.array([z_plane])
    X = axis(nx)[None, None, :]
    Y = axis(ny)[None, :, None]
    Z = axis(nz)[zs][:, None, None]
    idx = (zs[:, None, None].astype(np.int64) * ny + np.arange(ny)[None, :, None]) * nx + np.arange(nx)[None, None, :]
    X, Y, Z = np.broadcast_arrays(X, Y, Z)
    return shell_intensity(X, Y, Z, seed, idx, perturb)


def slice_stack(nx: int, ny: int, slices: int, depth_vox: int, seed: int) -> np.ndarray:
    """A sparse axial stack: ``slices`` planes of an nx*ny*depth_vox phantom, sampled at the
    nearest-source positions a resample would read (C3: 128x128x29 -> 128^3)."""
    zpos = np.round(np.linspace(0, depth_vox - 1, slices)).astype(np.int64)
    out = np.empty((slices, ny, nx), dtype=np.uint8)
    for s, zp in enumerate(zpos):
        out[s] = shell_phantom(nx, ny, depth_vox, seed, z_plane=int(zp))[0]
    return out


def pick_seed_voxel(labels: np.ndarray, shape, seed: int, salt: int = 5, margin: int = 1):
    """A seeded interior white-matter voxel whose (2*margin+1)^3 neighbourhood is all white.

    labels: x-fastest uint8 material codes.  Returns 0-based (i, j, k).
    """
    nx, ny, nz = shape
    lab = labels.reshape(nz, ny, nx) == 1
    ok = lab.copy()
    for dz in range(-margin, margin + 1):
        for dy in range(-margin, margin + 1):
            for dx in range(-margin, margin + 1):
                ok &= np.roll(lab, (dz, dy, dx), axis=(0, 1, 2))
    if nz == 1:
        ok = lab.copy()
        for dy in range(-margin, margin + 1):
            for dx in range(-margin, margin + 1):
                ok &= np.roll(lab, (dy, dx), axis=(1, 2))
    # exclude the wrap-around border
    if nz > 1:
        ok[:margin] = ok[nz - margin:] = False
    ok[:, :margin] = ok[:, ny - margin:] = False
    ok[:, :, :margin] = ok[:, :, nx - margin:] = False
    cand = np.flatnonzero(ok.ravel())
    if cand.size == 0:
        cand = np.flatnonzero(lab.ravel())
    if cand.size == 0:
        raise ValueError("phantom has no white matter")
    r = int(_stream(seed, salt, 1)[0] % np.uint64(cand.size))
    v = int(cand[r])
    return v % nx, (v // nx) % ny, v // (nx * ny)

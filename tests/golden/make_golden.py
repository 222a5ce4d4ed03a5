"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py

Outputs (committed, small):
  kat_reference.npz  the reference's own KAT inputs (mt19937_64 sequences of
                     test_expact.cpp / test_stencil.cpp / acceptance.cpp) with the
                     reference library's outputs and the dense-oracle outputs
                     (gen_golden.cpp, compiled against the reference by oracle/Makefile)
  material.npz       classify / resample / diffusion_from_materials KATs
                     (test_imaging.cpp:48-58, 131-191 shapes) and a 29-slice stack
  runs.npz           exponential-Euler trajectories of seeded shell phantoms computed by
                     gliosim::step / gliosim::run, plus the port's (s, m, terms) logs
"""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Port, Ref, build_ref, read_records  # noqa: E402
from paper_2402_02273_b200 import phantom  # noqa: E402


def kat_reference():
    build_ref()
    gen = os.path.join(ROOT, "oracle", "_ref", "gen_golden")
    tmp = "/tmp/gliosim_golden.bin"
    subprocess.check_call([gen, tmp])
    rec = read_records(tmp)
    np.savez_compressed(os.path.join(HERE, "kat_reference.npz"), **rec)
    print("kat_reference.npz:", len(rec), "arrays")


def material(ref: Ref):
    out = {"classify": np.array([ref.classify(v) for v in range(256)], dtype=np.uint8)}
    # test_imaging.cpp:131-162 brute-force nearest source: 1-D stacks of src pixels alternating
    # 0 / 100, resampled onto n points.
    for src in range(1, 8):
        px = np.array([0 if s % 2 == 0 else 100 for s in range(src)], dtype=np.uint8)
        for n in range(1, 8):
            out[f"nn.{src}.{n}"] = ref.resample(px, src, 1, 1, (n, 1, 1))
    # C3-shaped sparse stack at small size: 24x20 in-plane, 29 slices -> 24x20x40 grid
    stack = phantom.slice_stack(24, 20, 29, 40, seed=3)
    out["stack29"] = stack.ravel()
    out["stack29.labels"] = ref.resample(stack.ravel(), 24, 20, 29, (24, 20, 40))
    # down- and up-sampling in x/y as well
    out["stack29.labels_xy"] = ref.resample(stack.ravel(), 24, 20, 29, (17, 31, 9))
    labels = out["stack29.labels"]
    out["stack29.d"] = ref.diffusion_from_labels(labels, (24, 20, 40))
    np.savez_compressed(os.path.join(HERE, "material.npz"), **out)
    print("material.npz:", len(out), "arrays")


RUNS = [
    # name, shape, seed, sigma_vox, rho, tau, tol, steps, perturb, mask_seed, h_override
    ("r16", (16, 16, 16), 11, 3.0, 0.025, 33.5, 1e-8, 8, 0.0, True, None),
    ("r2d", (40, 36, 1), 12, 4.0, 0.025, 33.5, 1e-8, 4, 0.0, True, 200.0 / 255.0),
    ("rtau", (12, 10, 8), 13, 2.0, 0.1, 335.0, 1e-8, 4, 0.0, True, 5.0),
    ("rs9", (14, 12, 10), 17, 2.0, 0.025, 33.5, 1e-8, 3, 0.0, True, 1.0),
    ("r4rho", (20, 18, 16), 14, 3.0, 0.1, 33.5, 1e-8, 5, 0.1, True, None),
    ("runmasked", (10, 9, 7), 15, 2.0, 0.025, 33.5, 1e-10, 3, 0.0, False, None),
    ("rflat", (9, 1, 1), 16, 1.0, 0.3, 33.5, 1e-8, 3, 0.0, True, 200.0 / 8.0),
]


def make_case(shape, seed, sigma, perturb, mask, h_override, ref: Ref):
    nx, ny, nz = shape
    h = h_override if h_override else 200.0 / (max(shape) - 1)
    if nz == 1 and ny > 1:
        inten = phantom.shell_phantom(nx, ny, 2 * max(nx, ny), seed, perturb, z_plane=max(nx, ny))
    else:
        inten = phantom.shell_phantom(nx, ny, nz, seed, perturb)
    labels = np.array([ref.classify(int(v)) for v in range(256)], dtype=np.uint8)[inten.ravel()]
    if nx * ny * nz < 16:
        labels[:] = 1
        labels[nx // 2] = 2
    d = ref.diffusion_from_labels(labels, shape)
    i, j, k = phantom.pick_seed_voxel(labels, shape, seed, margin=1 if min(nx, ny) > 4 else 0)
    center = (i * h, j * h, k * h)
    width = 1.0 / (2.0 * (sigma * h) ** 2)
    u0 = ref.seed_initial(shape, h, 1.0, width, center, d if mask else None)
    return h, labels, d, center, width, u0


def runs(ref: Ref, port: Port):
    out = {}
    for name, shape, seed, sigma, rho, tau, tol, steps, perturb, mask, hov in RUNS:
        h, labels, d, center, width, u0 = make_case(shape, seed, sigma, perturb, mask, hov, ref)
        states = [u0]
        u = u0
        for _ in range(steps):
            u = ref.step(shape, h, d, u, rho, tau, tol)
            states.append(u)
        t0 = 150.0
        uf, metrics, _ = ref.run(shape, h, d, u0, steps, rho, t0, t0 + steps * tau, tol, center)
        assert np.array_equal(uf, states[-1]), name
        op = port.stencil(shape, h, d)
        s_m_terms = []
        for n in range(steps):
            _, log = port.step(op, states[n], rho, tau, tol)
            s_m_terms.append([log.s, log.m, log.total_terms])
        p = name + "."
        out[p + "shape"] = np.array(shape, dtype=np.int64)
        out[p + "params"] = np.array([h, rho, tau, tol, width, *center], dtype=np.float64)
        out[p + "labels"] = labels
        out[p + "states"] = np.stack(states)
        out[p + "metrics"] = metrics
        out[p + "log"] = np.array(s_m_terms, dtype=np.int64)
        print(name, shape, "s,m,terms per step:", s_m_terms)
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **out)
    print("runs.npz:", len(out), "arrays")


def main():
    kat_reference()
    ref = Ref()
    material(ref)
    runs(ref, Port())


if __name__ == "__main__":
    main()

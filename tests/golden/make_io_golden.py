"""Generate the file-format golden fixtures (tests/golden/io/) with the UNMODIFIED
reference library (oracle/_ref, built from /root/reference/proj by oracle/Makefile).

    python tests/golden/make_io_golden.py

Files (all written by the reference's own writers, vtk.cpp:59-157, imaging.cpp:166-173):
  layout.vtk         2x2x1 field of test_io.cpp:51-69
  mixed.vtk          3x4x2 field, origin (1,-2,0.125), h = 200/49, values that stress %.17g
                     (thirds, tenths, 1e-17, subnormals, -0.0, huge/tiny magnitudes), plus labels
  mixed_values.npy   the doubles of mixed.vtk (exact)
  mixed_labels.npy   its labels
  metrics.csv        a 6-row series; metrics_series.npz holds its inputs
  labels.raw         write_label_volume of a 5x4x3 volume; labels.npy holds it
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Ref  # noqa: E402

OUT = os.path.join(HERE, "io")


def stress_values(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.uniform(-1, 1, n)
    special = [1.0 / 3, 0.1, 1e-17, 5e-324, 2.2250738585072014e-308, -0.0, 1.7976931348623157e308,
               123456789012345678.0, 1e16, 1e17, 9.999999999999999e-5, 1e-4, 0.5, 2.0 / 3, -7.25e-300]
    v[:len(special)] = special
    return v


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = Ref()
    ref.write_vtk(os.path.join(OUT, "layout.vtk"), np.array([0.0, 0.5, 0.25, 1.0]), (2, 2, 1), 1.5)
    vals = stress_values(24, 17)
    labels = np.random.default_rng(3).integers(0, 4, 24).astype(np.uint8)
    ref.write_vtk(os.path.join(OUT, "mixed.vtk"), vals, (3, 4, 2), 200.0 / 49.0, (1.0, -2.0, 0.125), labels)
    np.save(os.path.join(OUT, "mixed_values.npy"), vals)
    np.save(os.path.join(OUT, "mixed_labels.npy"), labels)
    rng = np.random.default_rng(5)
    steps = np.arange(6, dtype=np.int32)
    times = 150.0 + 33.5 * steps
    m4 = rng.uniform(0, 1, (6, 4))
    m4[0] = [2.5, 0.0625, -0.5, 0.0]
    ref.write_metrics_csv(os.path.join(OUT, "metrics.csv"), steps, times, m4)
    np.savez(os.path.join(OUT, "metrics_series.npz"), steps=steps, times=times, m4=m4)
    lab = np.random.default_rng(9).integers(0, 4, 60).astype(np.uint8)
    ref.write_label_volume(os.path.join(OUT, "labels.raw"), lab, (5, 4, 3))
    np.save(os.path.join(OUT, "labels.npy"), lab)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()

"""CPU check of the full-run parity harness (tests/fullrun.py) itself: a stand-in operator
that steps with the C restatement must pass every gate against the compiled reference, and
a stand-in that perturbs one step must fail them.  No GPU."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import fullrun as FR  # noqa: E402


class _Info:
    def __init__(self, log):
        self.s, self.m, self._t = log.s, log.m, log.stage_terms()

    def stage_terms(self):
        return list(self._t)


class _Grid:
    def __init__(self, shape, h):
        self.shape, self.h = shape, h


class FakeOp:
    """Steps with the oracle; `bad_step` adds a 1e-9 relative kick after that step."""

    def __init__(self, port, shape, h, d, bad_step=None):
        self.port, self.grid = port, _Grid(shape, h)
        self.op_o = port.stencil(shape, h, d)
        self.u = None
        self.k = 0
        self.bad_step = bad_step

    def set_state(self, u):
        self.u = np.array(u, copy=True)
        self.k = 0

    def get_state(self):
        return self.u.copy()

    def run_resident(self, n, rho, tau, tol, origin=(0.0, 0.0, 0.0), center=(0.0, 0.0, 0.0), front=0.1,
                     metrics=True, infos=False):
        class M:
            pass
        mets, inf = [], []

        def node():
            m = M()
            m.total_mass, m.max_density, m.min_density, m.radius = self.port.compute_metrics(
                self.u, self.grid.shape, self.grid.h, center, front)
            return m
        mets.append(node())
        for _ in range(n):
            self.u, log = self.port.step(self.op_o, self.u, rho, tau, tol)
            self.k += 1
            if self.k == self.bad_step:
                self.u = self.u * (1.0 + 1e-9)
            inf.append(_Info(log))
            mets.append(node())
        return mets, inf


def _case(port):
    shape = (12, 10, 8)
    h = 200.0 / 11
    rng = np.random.default_rng(3)
    labels = rng.choice(np.array([0, 1, 1, 1, 2, 3], dtype=np.uint8), size=int(np.prod(shape)))
    d = port.diffusion_from_labels(labels)
    center = (5 * h, 4 * h, 3 * h)
    u0 = port.seed_initial(shape, h, 1.0, 1.0 / (2 * (2 * h) ** 2), center, d)
    return shape, h, labels, d, center, u0


def test_harness_passes_the_oracle(port, ref):
    shape, h, labels, d, center, u0 = _case(port)
    op = FakeOp(port, shape, h, d)
    rec = FR.full_run_parity("fake", op, labels, u0, 6, 0.025, 33.5, 1e-8, center, port, ref, threads=3,
                             log=lambda *_: None)
    FR.assert_record(rec)
    assert rec["final_rel_l2_vs_reference"] == 0.0  # the port is bitwise the reference
    assert len(rec["per_step"]) == 6 and [r["step"] for r in rec["per_step"]] == list(range(1, 7))


def test_harness_catches_a_perturbed_step(port, ref):
    shape, h, labels, d, center, u0 = _case(port)
    op = FakeOp(port, shape, h, d, bad_step=3)
    rec = FR.full_run_parity("fake", op, labels, u0, 6, 0.025, 33.5, 1e-8, center, port, ref, threads=3,
                             log=lambda *_: None)
    with pytest.raises(AssertionError):
        FR.assert_record(rec)
    assert rec["per_step"][2]["rel_l2"] > 1e-10

"""Parity at BASELINE.json's full size (C4, 256^3 = 16.7 M voxels), on the GPU.

The oracle is single-threaded C, so one exponential-Euler step of it at 256^3 takes
tens of seconds: these tests use one step plus size-independent properties.
* one C4 step: material map exact; (s, m) and the terms of every stage exact; u within
  the per-step bar (relative L2 1e-10) of the oracle; and, given the device's two
  order-dependent sums, bit-identical to it;
* expmv is homogeneous bit for bit: expmv(t, A, 2b) == 2 expmv(t, A, b) (scaling by two
  is exact and leaves every termination decision unchanged);
* with uniform D the stencil's columns sum to zero, so expmv conserves mass;
* the semigroup property expmv(t1 + t2) = expmv(t2, expmv(t1)) holds within tolerance.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c4():
    import bench
    from paper_2402_02273_b200 import workloads as W
    w = W.get("C4")
    data, dims, labels = bench.build_case(w)
    op = bench.make_operator(w, data, dims)
    u0 = bench.initial_state(w, op, labels)
    yield w, op, labels, u0
    op.close()


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_c4_step_matches_oracle(c4, port):
    from paper_2402_02273_b200 import gliosim as G
    from paper_2402_02273_b200 import workloads as W
    w, op, labels, u0 = c4
    assert np.array_equal(op.labels(), labels)  # K1 at full size
    d = port.diffusion_from_labels(labels)
    op_o = port.stencil((w.nx, w.ny, w.nz), w.h, d)
    assert op.one_norm() == port.one_norm(op_o)  # exact 1-norm
    got, info = G.step(op, u0, w.rho, w.tau, W.TOL, info=True)
    want, log = port.step(op_o, u0, w.rho, w.tau, W.TOL, bnorm=info.bnorm, coln=info.coln)
    assert (info.s, info.m) == (log.s, log.m)
    assert info.stage_terms() == log.stage_terms()
    assert np.array_equal(got, want)
    plain, log2 = port.step(op_o, u0, w.rho, w.tau, W.TOL)
    assert rel_l2(got, plain) <= 1e-10
    assert info.total_terms == log2.total_terms


def test_c4_expmv_is_exactly_homogeneous(c4):
    from paper_2402_02273_b200 import gliosim as G
    w, op, labels, u0 = c4
    y1 = G.expmv(w.tau, op, u0, 1e-8)
    y2 = G.expmv(w.tau, op, 2.0 * u0, 1e-8)
    assert np.array_equal(y2, 2.0 * y1)


def test_c4_uniform_diffusion_conserves_mass_and_semigroup(c4):
    from paper_2402_02273_b200 import gliosim as G
    w, op, labels, u0 = c4
    grid = G.Grid(w.nx, w.ny, w.nz, w.h)
    with G.assemble_diffusion(grid, np.full(grid.num_points(), 0.13)) as a:
        y = G.expmv(200.0, a, u0, 1e-10)
        assert abs(y.sum() - u0.sum()) <= 1e-9 * np.abs(u0).sum()
        assert y.min() >= -1e-12 * u0.max() and y.max() <= u0.max() * (1 + 1e-12)  # max principle
        y_ab = G.expmv(120.0, a, G.expmv(80.0, a, u0, 1e-12), 1e-12)
        assert rel_l2(y_ab, y) <= 1e-9


def test_c5_batched_members_match_oracle(port):
    """C5 at full member size (128^3): three members of the real ensemble (lowest, highest and
    a middle rho) advanced two batched steps (gs_run_ensemble, 16 groups, the members taken from
    the queue) -- every member and step bitwise against the oracle given that member's device
    sums, terms per stage exact, and within the per-step bar without the sums."""
    from paper_2402_02273_b200 import ensemble as E
    from paper_2402_02273_b200 import workloads as W
    w = W.get("C5")
    rhos = [W.member_rho(w, mb) for mb in range(w.members)]
    pick = sorted({int(np.argmin(rhos)), int(np.argmax(rhos)), w.members // 2})
    runner = E.EnsembleRunner(w, pick)
    try:
        runner.reset()
        from paper_2402_02273_b200 import gliosim as G
        _, infos = G.run_ensemble(runner.ops, 2, runner.rhos, w.tau, W.TOL, metrics=False, infos=True)
        for i, (op, u0, rho) in enumerate(zip(runner.ops, runner.u0, runner.rhos)):
            op_o = port.stencil((w.nx, w.ny, w.nz), w.h, port.diffusion_from_labels(op.labels()))
            u = u0
            for q in range(2):
                inf = infos[i][q]
                want, log = port.step(op_o, u, rho, w.tau, W.TOL, bnorm=inf.bnorm, coln=inf.coln)
                assert inf.stage_terms() == log.stage_terms(), (i, q)
                plain, _ = port.step(op_o, u, rho, w.tau, W.TOL)
                assert rel_l2(want, plain) <= 1e-10
                u = want
            assert np.array_equal(op.get_state(), u), i
    finally:
        runner.close()

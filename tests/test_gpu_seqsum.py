"""The reference's two order-dependent sums, reproduced bit for bit on the GPU
(paper_2402_02273_b200/csrc/gs_seqsum.cuh):

* ||b||_1 = sum |b_i| left to right (expact.cpp:20-24, called at :110);
* the bordered column sum sum_{b_i != 0} |b_i / gamma| in row order (sparse.cpp:36-38 on the
  operator expact.cpp:131-142 builds).

np.cumsum is a sequential left-to-right accumulation, so its last element is the reference's
value.  The vectors are built to stress the parallel emulation: values spanning hundreds of
binades (Gaussian tails), exact rounding ties (multiples of 1/8 against sums in binades whose
ulp is 1/4 or 1/2), subnormals, long zero runs, and sizes around the tile size.  phi1v reports
both sums in its step info; a 2-D C2-sized Gaussian also checks the whole step bitwise against
the oracle with no device sums passed in.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu

TILE = 512 * 8


def seq_sum(x):
    return float(np.cumsum(np.abs(x))[-1]) if len(x) else 0.0


def _vectors(n, rng):
    out = {}
    i = np.arange(n, dtype=np.float64)
    c = n * rng.uniform(0.3, 0.7)
    w = max(n / 40.0, 1.0)
    out["gauss_tails"] = np.exp(-((i - c) / w) ** 2 * 0.5) * rng.choice([-1.0, 1.0], n)
    out["geometric"] = np.exp(np.linspace(-700.0, 2.0, n)) * (1 + 0.1 * rng.random(n))
    out["ties"] = rng.integers(0, 64, n) / 8.0
    out["ties_scaled"] = rng.integers(0, 9, n) * 2.0 ** rng.integers(-60, -50, n)
    sub = rng.random(n) * 2.0 ** -1060
    sub[rng.random(n) < 0.5] = 0.0
    out["subnormal"] = sub
    z = rng.standard_normal(n) * np.exp(rng.uniform(-300, 0, n))
    z[rng.random(n) < 0.7] = 0.0
    out["sparse_wide"] = z
    out["descending"] = np.exp(np.linspace(5.0, -700.0, n))
    return out


@pytest.mark.parametrize("shape", [(8, 4, 1), (16, 16, 16), (64, 64, 1), (48, 33, 20), (96, 96, 32)])
def test_sequential_sums_bitwise(shape, port):
    from paper_2402_02273_b200 import gliosim as G
    n = int(np.prod(shape))
    rng = np.random.default_rng(n)
    d = np.full(n, 0.13)
    d[rng.random(n) < 0.1] = 0.0
    h = 0.5
    with G.StencilOperator.from_diffusion(G.Grid(*shape, h), d) as op:
        anorm = op.one_norm()
        for name, b in _vectors(n, rng).items():
            b = np.ascontiguousarray(b, dtype=np.float64)
            _, info = G.phi1v(0.7, op, b, 1e-8, info=True)
            want = seq_sum(b)
            assert info.bnorm == want, (name, info.bnorm, want, info.bnorm - want)
            if info.branch == 0:
                gamma = want / anorm
                assert info.gamma == gamma
                bg = np.where(b != 0.0, b / gamma, 0.0)
                assert info.coln == seq_sum(bg), (name, info.coln, seq_sum(bg))


def test_non_finite_sums(port):
    """NaN anywhere makes the sequential sum NaN, +-inf (without NaN) makes it inf; the step
    then behaves as the oracle's (its own tests cover the error path)."""
    from paper_2402_02273_b200 import gliosim as G
    shape = (32, 16, 4)
    n = int(np.prod(shape))
    with G.StencilOperator.from_diffusion(G.Grid(*shape, 0.5), np.full(n, 0.13)) as op:
        for bad, want in ((np.inf, np.inf), (-np.inf, np.inf), (np.nan, None)):
            b = np.linspace(0.0, 1.0, n)
            b[n // 3] = bad
            try:
                _, info = G.phi1v(0.7, op, b, 1e-8, info=True)
            except G.NumericError:
                continue
            if want is None:
                assert np.isnan(info.bnorm)
            else:
                assert info.bnorm == want


def test_c2_step_bitwise_without_device_sums(port):
    """C2's first step is the case where one ulp of ||b||_1 moves u by 1e-10: with the
    sequential sums the GPU step equals the oracle's bit for bit, no device sums passed."""
    import bench
    from paper_2402_02273_b200 import workloads as W
    from paper_2402_02273_b200 import gliosim as G
    w = W.get("C2")
    data, dims, labels = bench.build_case(w)
    with bench.make_operator(w, data, dims) as op:
        u0 = bench.initial_state(w, op, labels)
        got, info = G.step(op, u0, w.rho, w.tau, W.TOL, info=True)
    op_o = port.stencil((w.nx, w.ny, w.nz), w.h, port.diffusion_from_labels(labels))
    want, log = port.step(op_o, u0, w.rho, w.tau, W.TOL)
    assert info.bnorm == log.bnorm and info.coln == log.coln
    assert info.stage_terms() == log.stage_terms()
    assert np.array_equal(got, want)

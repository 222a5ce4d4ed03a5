"""Races by repetition.  compute-sanitizer is closed on the GPU pool (runs under it have left
GPUs needing a reset), so the asynchronous machinery is checked by its observable effect: a
race between the TMA ring's producer and consumers, the mbarrier phases, the async-proxy
fences, the grid / group / cluster barriers, the per-term max slots or the seqsum tickets
would make repeated launches disagree or disagree with the oracle.  Each path runs the same
multi-step launch many times; every result must equal the oracle's bit for bit."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPEATS = 25


@pytest.fixture(scope="module")
def G():
    from paper_2402_02273_b200 import gliosim
    return gliosim


def _field(shape, seed):
    rng = np.random.default_rng(seed)
    n = int(np.prod(shape))
    d = np.array([0.0, 0.13, 0.013, 0.05])[rng.integers(0, 4, n)]
    u = np.zeros(n)
    u[rng.integers(0, n, 60)] = rng.uniform(0.2, 1.0, 60)
    u[d == 0.0] = 0.0
    return d, u


def _oracle(port, shape, h, d, u, steps, rho=0.025):
    op_o = port.stencil(shape, h, d)
    for _ in range(steps):
        u, _ = port.step(op_o, u, rho, 33.5, 1e-8)
    return u


@pytest.mark.parametrize("path,shape", [("tma2", (48, 32, 20)), ("tma3", (48, 32, 20)), ("l1", (40, 24, 18)),
                                        ("cluster", (32, 32, 32)), ("thin", (64, 48, 1)),
                                        ("flat2d", (200, 190, 1))])
def test_repeated_runs_identical(G, port, path, shape, monkeypatch):
    if path != "cluster":
        monkeypatch.setenv("GS_NO_CLUSTER", "1")
    if path != "flat2d":
        monkeypatch.setenv("GS_NO_2D", "1")
    if path == "l1":
        monkeypatch.setenv("GS_DISABLE_TMA", "1")
    if path == "tma3":
        monkeypatch.setenv("GS_FUSE", "3")
    d, u0 = _field(shape, sum(shape))
    h = 0.5
    want = _oracle(port, shape, h, d, u0, 3)
    with G.assemble_diffusion(G.Grid(*shape, h=h), d) as op:
        assert op.uses_cluster() == (path == "cluster")
        assert op.uses_flat2d() == (path == "flat2d")
        for _ in range(REPEATS):
            op.set_state(u0)
            op.run_resident(3, 0.025, 33.5, 1e-8, metrics=True, infos=True)
            assert np.array_equal(op.get_state(), want)


def test_repeated_batched_ensemble_identical(G, port):
    shapes = [(48, 32, 20), (32, 32, 24), (64, 16, 16), (48, 32, 20), (32, 16, 32)]
    rhos = [0.025, 0.05, 0.01, 0.1, 0.03]
    ops, u0s, wants = [], [], []
    try:
        for k, (s, rho) in enumerate(zip(shapes, rhos)):
            d, u = _field(s, 100 + k)
            ops.append(G.assemble_diffusion(G.Grid(*s, h=0.5), d))
            u0s.append(u)
            wants.append(_oracle(port, s, 0.5, d, u, 2, rho))
        for rep in range(REPEATS):
            for op, u in zip(ops, u0s):
                op.set_state(u)
            G.run_ensemble(ops, 2, rhos, 33.5, 1e-8, metrics=True, infos=True, groups=2 + rep % 3)
            for op, want in zip(ops, wants):
                assert np.array_equal(op.get_state(), want), rep
    finally:
        for op in ops:
            op.close()


def test_two_contexts_two_threads(G, port):
    """Two operators stepped from two host threads at once (own streams, concurrent kernels)."""
    cases = [((48, 32, 20), 1), ((40, 32, 16), 2)]
    items = []
    for shape, seed in cases:
        d, u = _field(shape, seed)
        items.append((shape, d, u, _oracle(port, shape, 0.5, d, u, 2)))
    ops = [G.assemble_diffusion(G.Grid(*s, h=0.5), d) for s, d, _, _ in items]
    errors = []

    def work(op, u0, want):
        try:
            for _ in range(REPEATS):
                op.set_state(u0)
                op.run_resident(2, 0.025, 33.5, 1e-8, metrics=False)
                if not np.array_equal(op.get_state(), want):
                    errors.append("mismatch")
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    try:
        th = [threading.Thread(target=work, args=(op, it[2], it[3])) for op, it in zip(ops, items)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    finally:
        for op in ops:
            op.close()
    assert not errors, errors[:3]

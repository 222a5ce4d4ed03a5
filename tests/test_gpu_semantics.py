"""Boundary semantics of the drop-in against the reference's API contract
(/root/reference/proj/include/gliosim/integrator.hpp:59-77, SPEC.md's concurrency model):

* step() / phi1v() / expmv() / apply() have value semantics and take the operator by const
  reference: they must not disturb the resident state a run works on;
* concurrent step() calls on one operator give the serial results (the context serialises);
* a wrong vector length raises what the reference's first use of the vector raises
  (SparseOperator::apply, sparse.cpp:44-46, for step);
* run()'s StepWatcher / RangeWarning fire after each step, while the run is in progress
  (integrator.cpp:128-131), so a progress hook is live;
* compute_metrics places points with the operator's grid (integrator.cpp:65-89).
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = {"cluster": (24, 16, 16), "multikernel": (48, 32, 20)}


@pytest.fixture(scope="module")
def G():
    from paper_2402_02273_b200 import gliosim
    return gliosim


def _case(shape, seed=3):
    rng = np.random.default_rng(seed)
    n = int(np.prod(shape))
    d = np.array([0.0, 0.13, 0.013, 0.05])[rng.integers(0, 4, n)]
    u0 = np.zeros(n)
    u0[rng.integers(0, n, 60)] = rng.uniform(0.2, 1.0, 60)
    u0[d == 0.0] = 0.0
    return d, u0, rng


def _path(path, monkeypatch):
    if path == "multikernel":
        monkeypatch.setenv("GS_NO_CLUSTER", "1")


@pytest.mark.parametrize("path", ["cluster", "multikernel"])
def test_value_calls_leave_resident_state_intact(G, port, path, monkeypatch):
    _path(path, monkeypatch)
    shape = SHAPES[path]
    d, u0, rng = _case(shape)
    h = 0.5
    op_o = port.stencil(shape, h, d)
    other = rng.uniform(0.0, 1.0, u0.size)
    with G.assemble_diffusion(G.Grid(*shape, h=h), d) as op:
        assert op.uses_cluster() == (path == "cluster")
        op.set_state(u0)
        op.run_resident(4, 0.025, 33.5, 1e-8, metrics=False)
        straight = op.get_state()
        op.set_state(u0)
        op.run_resident(2, 0.025, 33.5, 1e-8, metrics=False)
        mid = op.get_state()
        got = G.step(op, other, 0.025, 33.5, 1e-8)                 # value semantics...
        want, _ = port.step(op_o, other, 0.025, 33.5, 1e-8)
        assert np.array_equal(got, want)                           # ...bitwise the reference's step
        G.phi1v(10.0, op, other, 1e-8)
        G.expmv(10.0, op, other, 1e-8)
        op.apply(other)
        assert np.array_equal(op.get_state(), mid)                 # resident state untouched
        op.run_resident(2, 0.025, 33.5, 1e-8, metrics=False)
        assert np.array_equal(op.get_state(), straight)            # and the run continues as if alone


def test_step_ensemble_host_leaves_resident_states_intact(G, port):
    shapes = [(48, 32, 20), (32, 32, 24)]
    ops, mids, ins = [], [], []
    try:
        for k, shape in enumerate(shapes):
            d, u0, rng = _case(shape, seed=10 + k)
            op = G.assemble_diffusion(G.Grid(*shape, h=0.5), d)
            ops.append(op)
            op.set_state(u0)
            op.run_resident(1, 0.025, 33.5, 1e-8, metrics=False)
            mids.append(op.get_state())
            ins.append(rng.uniform(0.0, 1.0, u0.size))
        outs, _ = G.step_ensemble_host(ops, ins, [0.025, 0.05], 33.5, 1e-8)
        for op, mid, u, o, rho, shape in zip(ops, mids, ins, outs, [0.025, 0.05], shapes):
            assert np.array_equal(op.get_state(), mid)
            assert np.array_equal(o, G.step(op, u, rho, 33.5, 1e-8))
    finally:
        for op in ops:
            op.close()


def test_step_ensemble_host_rejects_bad_outputs(G):
    shape = (32, 16, 8)
    d, u0, _ = _case(shape)
    with G.assemble_diffusion(G.Grid(*shape, h=0.5), d) as op:
        n = u0.size
        for bad in (np.empty(n, dtype=np.float32), np.empty(n - 1), np.empty((2, n))[:, 0], np.empty(n)[::1].copy()[:-1]):
            with pytest.raises(ValueError, match="output"):
                G.step_ensemble_host([op], [u0], [0.025], 33.5, 1e-8, outs=[bad])
        ro = np.empty(n)
        ro.setflags(write=False)
        with pytest.raises(ValueError, match="output"):
            G.step_ensemble_host([op], [u0], [0.025], 33.5, 1e-8, outs=[ro])
        with pytest.raises(ValueError, match="one output"):
            G.step_ensemble_host([op], [u0], [0.025], 33.5, 1e-8, outs=[])


def test_concurrent_steps_on_one_operator(G):
    """Two host threads stepping the same operator (ctypes releases the GIL): every result
    equals the serial one bit for bit."""
    shape = (48, 32, 20)
    d, u0, rng = _case(shape)
    inputs = [rng.uniform(0.0, 1.0, u0.size) for _ in range(6)]
    with G.assemble_diffusion(G.Grid(*shape, h=0.5), d) as op:
        serial = [G.step(op, u, 0.025, 33.5, 1e-8) for u in inputs]
        results = [None] * len(inputs)

        def worker(idx):
            for _ in range(3):
                for i in idx:
                    results[i] = G.step(op, inputs[i], 0.025, 33.5, 1e-8)

        th = [threading.Thread(target=worker, args=(list(range(k, len(inputs), 2)),)) for k in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for a, b in zip(results, serial):
            assert np.array_equal(a, b)


def test_step_length_mismatch_message(G):
    shape = (16, 8, 4)
    d, u0, _ = _case(shape)
    with G.assemble_diffusion(G.Grid(*shape, h=0.5), d) as op:
        with pytest.raises(ValueError, match=r"^SparseOperator::apply: vector length 5 != dim 512$"):
            G.step(op, np.ones(5), 0.025, 33.5, 1e-8)
        with pytest.raises(ValueError, match="phi1v: vector length does not match operator dimension"):
            G.phi1v(1.0, op, np.ones(5), 1e-8)
        with pytest.raises(ValueError, match="expmv: vector length does not match operator dimension"):
            G.expmv(1.0, op, np.ones(5), 1e-8)


@pytest.mark.parametrize("path", ["cluster", "multikernel"])
def test_run_hooks_fire_live(G, path, monkeypatch):
    """on_step sees each step's state while the run is in progress (the state after step k is
    resident when the hook for step k fires); on_range fires for the steps that leave
    [-0.01, 1.01] -- here an explicit logistic term with rho tau > 3, which overshoots."""
    _path(path, monkeypatch)
    shape = SHAPES[path]
    d, _, _ = _case(shape)
    d = np.where(d > 0.0, d, 0.05)  # no dead voxels: a uniform u has A u = 0 (row-constant D)
    u0 = np.full(d.size, 0.5)       # 0.5 + tau rho 0.25 = 1.34: the explicit logistic term overshoots
    h = 0.5
    steps = 6
    rho = 0.1
    grid = G.Grid(*shape, h=h)
    cfg = G.SimConfig(nx=shape[0], ny=shape[1], nz=shape[2], h=h, rho=rho, t0=150.0,
                      t_end=150.0 + steps * 33.5, num_steps=steps, exp_tol=1e-8, seed_center=(1.0, 1.0, 1.0))
    with G.assemble_diffusion(grid, d) as op:
        op.set_state(u0)
        want = []
        for _ in range(steps):
            op.run_resident(1, rho, 33.5, 1e-8, metrics=False)
            want.append(op.get_state())
        seen, states, ranges = [], [], []

        def on_step(m):
            seen.append(m.step)
            states.append(op.get_state())

        res = G.run(cfg, op, u0, on_step=on_step, on_range=lambda k, lo, hi: ranges.append((k, lo, hi)))
    assert seen == list(range(1, steps + 1))
    for k in range(steps):
        assert np.array_equal(states[k], want[k]), k
    expect = [m.step for m in res.metrics[1:] if m.min_density < -0.01 or m.max_density > 1.01]
    assert [r[0] for r in ranges] == expect and expect  # the overshoot happens, and is reported live


def test_run_metrics_use_the_grid_origin(G, port):
    """SimConfig.origin and the operator grid's origin differ: compute_metrics follows the
    DiffusionField's grid (integrator.cpp:65-89), i.e. the operator's."""
    shape = (32, 16, 16)
    d, u0, _ = _case(shape)
    h = 0.5
    gorigin = (3.0, -2.0, 1.5)
    grid = G.Grid(*shape, h=h, origin=gorigin)
    center = (9.0, 2.0, 5.0)
    cfg = G.SimConfig(nx=shape[0], ny=shape[1], nz=shape[2], h=h, origin=(0.0, 0.0, 0.0), rho=0.025, t0=150.0,
                      t_end=150.0 + 2 * 33.5, num_steps=2, exp_tol=1e-8, seed_center=center)
    with G.assemble_diffusion(grid, d) as op:
        res = G.run(cfg, op, u0)
    want = port.compute_metrics(u0, shape, h, center, 0.1, origin=gorigin)
    got = res.metrics[0]
    assert got.radius == want[3]
    assert got.max_density == want[1] and got.min_density == want[2]

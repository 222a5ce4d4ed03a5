"""Multi-rank host logic of the C5 ensemble (replicas: members partitioned over ranks, one
gather at the end), exercised with world_size 2 over gloo on the CPU."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_02273_b200 import ensemble as E


def test_members_partition_is_exact_and_balanced():
    for world in range(1, 9):
        seen = []
        sizes = []
        for r in range(world):
            m = E.members_for_rank(64, r, world)
            seen += m
            sizes.append(len(m))
        assert sorted(seen) == list(range(64))
        assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    steps = 3
    res = []
    for mb in E.members_for_rank(8, rank, world):
        met = np.full((steps + 1, 4), float(mb))
        res.append(E.MemberResult(mb, 0.025, steps, met, np.full(steps, 10 + mb), float(mb)))
    table, terms = E.gather_results(res, 8, steps, dist)
    if rank == 0:
        q.put((table, terms))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_over_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    table, terms = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for mb in range(8):
        assert np.all(table[mb] == mb)
        assert np.all(terms[mb] == 10 + mb)


@pytest.mark.gpu
def test_ensemble_members_match_single_runs():
    """Two members through the EnsembleRunner equal the same members run alone (and the oracle)."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    from oracle import Port
    from paper_2402_02273_b200 import workloads as W
    small = W.Workload("C5s", 32, 32, 32, 3, 2.0, 505, members=4)
    runner = E.EnsembleRunner(small, [1, 2])
    runner.reset()
    res = runner.run(3)
    port = Port()
    for r, op, u0, c, rho in zip(res, runner.ops, runner.u0, runner.centers, runner.rhos):
        d = port.diffusion_from_labels(op.labels())
        u, metrics, logs = port.run(port.stencil((32, 32, 32), small.h, d), u0, 3, rho, small.tau, W.TOL, c,
                                    with_logs=True)
        assert [lg.total_terms for lg in logs] == list(r.terms)
        np.testing.assert_allclose(r.metrics[:, 1], metrics[:, 1], rtol=1e-12)
        got = op.get_state()
        assert np.linalg.norm(got - u) / np.linalg.norm(u) <= 1e-10
    assert len({round(x, 12) for x in runner.rhos}) == 2
    runner.close()


def _random_members(port, shape, k, seed):
    """k members on one shape: random material fields, sparse initial states, distinct rho."""
    rng = np.random.default_rng(seed)
    n = int(np.prod(shape))
    out = []
    for i in range(k):
        d = np.array([0.0, 0.13, 0.013, 0.05])[rng.integers(0, 4, n)]
        u0 = np.zeros(n)
        u0[rng.integers(0, n, 60)] = rng.uniform(0.2, 1.0, 60)
        u0[d == 0.0] = 0.0
        out.append((d, u0, 0.025 * float(np.exp(rng.uniform(np.log(0.25), np.log(4.0))))))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("shape,groups", [((48, 32, 20), 2), ((48, 32, 20), 3), ((64, 48, 1), 2)])
def test_batched_ensemble_bitwise_vs_oracle(port, shape, groups):
    """gs_run_ensemble (one launch per kernel for all members; `groups` members at a time in the
    Taylor launch, taken from a queue): every member, every step bitwise against the oracle given
    that member's device sums, terms per stage equal, metrics of the final node exact."""
    from paper_2402_02273_b200 import gliosim as G
    h, tau, tol, steps = 2.0, 33.5, 1e-8, 3
    members = _random_members(port, shape, 5, sum(shape) + groups)
    ops = [G.assemble_diffusion(G.Grid(*shape, h=h), d) for d, _, _ in members]
    try:
        for op, (_, u0, _) in zip(ops, members):
            op.set_state(u0)
        centers = np.array([[10.0, 8.0, 4.0 * (i + 1)] for i in range(len(ops))])
        mets, infos = G.run_ensemble(ops, steps, [r for _, _, r in members], tau, tol, None, centers, 0.1,
                                     metrics=True, infos=True, groups=groups)
        for i, (op, (d, u0, rho)) in enumerate(zip(ops, members)):
            op_o = port.stencil(shape, h, d)
            u = u0
            for q in range(steps):
                inf = infos[i][q]
                u, log = port.step(op_o, u, rho, tau, tol, bnorm=inf.bnorm, coln=inf.coln)
                assert inf.stage_terms() == log.stage_terms(), (i, q)
            got = op.get_state()
            assert np.array_equal(got, u), i
            assert mets[i][steps].max_density == got.max()
            assert mets[i][steps].min_density == got.min()
    finally:
        for op in ops:
            op.close()


@pytest.mark.gpu
def test_batched_ensemble_reports_its_taylor_launch_times(port):
    """Kernel timing on member 0 brackets every step's batched Taylor launch with CUDA events
    (the C5 bench line's roofline): one launch per step, a positive total, results unchanged."""
    from paper_2402_02273_b200 import gliosim as G
    shape, h, tau, tol, steps = (48, 32, 20), 2.0, 33.5, 1e-8, 3
    members = _random_members(port, shape, 4, 77)
    ops = [G.assemble_diffusion(G.Grid(*shape, h=h), d) for d, _, _ in members]
    try:
        finals = []
        for timing in (False, True):
            for op, (_, u0, _) in zip(ops, members):
                op.set_state(u0)
            ops[0].set_kernel_timing(timing)
            G.run_ensemble(ops, steps, [r for _, _, r in members], tau, tol, metrics=False, infos=False, groups=2)
            if timing:
                ms, n = ops[0].kernel_times()["taylor"]
                assert n == steps and ms > 0.0
            finals.append([op.get_state() for op in ops])
        ops[0].set_kernel_timing(False)
        for a, b in zip(*finals):
            assert np.array_equal(a, b)
    finally:
        for op in ops:
            op.close()


@pytest.mark.gpu
def test_batched_ensemble_matches_sequential_runs(port, monkeypatch):
    """The batched ensemble against the same members run one after another (gs_run each): the
    same terms per stage, states equal up to the ulps of the per-CTA partial sums."""
    from paper_2402_02273_b200 import gliosim as G
    shape, h, tau, tol, steps = (48, 32, 20), 2.0, 33.5, 1e-8, 4
    members = _random_members(port, shape, 4, 99)
    finals = {}
    for mode in ("batched", "sequential"):
        if mode == "sequential":
            monkeypatch.setenv("GS_ENS_SEQUENTIAL", "1")
        ops = [G.assemble_diffusion(G.Grid(*shape, h=h), d) for d, _, _ in members]
        try:
            for op, (_, u0, _) in zip(ops, members):
                op.set_state(u0)
            _, infos = G.run_ensemble(ops, steps, [r for _, _, r in members], tau, tol, metrics=False, infos=True)
            finals[mode] = ([op.get_state() for op in ops],
                            [[infos[i][q].stage_terms() for q in range(steps)] for i in range(len(ops))])
        finally:
            for op in ops:
                op.close()
    (ub, tb), (us, ts) = finals["batched"], finals["sequential"]
    assert tb == ts
    for a, b in zip(ub, us):
        assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b)


@pytest.mark.gpu
def test_ensemble_mixed_shapes_fall_back_to_sequential(port):
    """Members the batched path cannot take together (here 2-D with 3-D) run one by one."""
    from paper_2402_02273_b200 import gliosim as G
    specs = [((48, 32, 20), 7), ((64, 48, 1), 8)]
    ops, refs = [], []
    try:
        for shape, seed in specs:
            (d, u0, rho), = _random_members(port, shape, 1, seed)
            op = G.assemble_diffusion(G.Grid(*shape, h=2.0), d)
            op.set_state(u0)
            ops.append(op)
            refs.append((shape, d, u0, rho))
        _, infos = G.run_ensemble(ops, 2, [r[3] for r in refs], 33.5, 1e-8, metrics=False, infos=True)
        for i, (op, (shape, d, u0, rho)) in enumerate(zip(ops, refs)):
            u = u0
            for q in range(2):
                u, _ = port.step(port.stencil(shape, 2.0, d), u, rho, 33.5, 1e-8, bnorm=infos[i][q].bnorm,
                                 coln=infos[i][q].coln)
            assert np.array_equal(op.get_state(), u)
    finally:
        for op in ops:
            op.close()


@pytest.mark.gpu
def test_ensemble_argument_errors(port):
    """Bad ensembles fail like the reference's run() does for one member (std::invalid_argument
    -> ValueError), before any device work."""
    from paper_2402_02273_b200 import gliosim as G
    (d, u0, rho), = _random_members(port, (48, 32, 20), 1, 3)
    with G.assemble_diffusion(G.Grid(48, 32, 20, h=2.0), d) as a, \
            G.assemble_diffusion(G.Grid(48, 32, 20, h=2.0), d) as b:
        a.set_state(u0)
        b.set_state(u0)
        with pytest.raises(ValueError, match="appears twice"):
            G.run_ensemble([a, a], 1, [rho, rho], 33.5, 1e-8)
        with pytest.raises(ValueError, match="tolerance"):
            G.run_ensemble([a, b], 1, [rho, rho], 33.5, 1.5)
        with pytest.raises(ValueError, match="one rho per member"):
            G.run_ensemble([a, b], 1, [rho], 33.5, 1e-8)
        with pytest.raises(ValueError, match="no members"):
            G.run_ensemble([], 1, [], 33.5, 1e-8)
        bare = G.StencilOperator(G.Grid(48, 32, 20, h=2.0))  # no operator set
        try:
            with pytest.raises(ValueError, match="member 1: operator not set"):
                G.run_ensemble([a, bare], 1, [rho, rho], 33.5, 1e-8)
        finally:
            bare.close()
        assert np.array_equal(a.get_state(), u0) and np.array_equal(b.get_state(), u0)


@pytest.mark.gpu
def test_batched_ensemble_heterogeneous_members(port):
    """Members of different 3-D shapes and the degenerate branches of phi1v in one batched
    call: b = 0 (u = 0: expact.cpp:111, the Taylor body returns before any group barrier),
    A = 0 (D = 0 everywhere: the small-norm branch, expact.cpp:114-121) and ordinary members,
    2 groups, several steps -- each member bitwise against the oracle given its device sums."""
    from paper_2402_02273_b200 import gliosim as G
    rng = np.random.default_rng(11)
    specs = []
    for shape, kind in [((48, 32, 20), "plain"), ((64, 48, 24), "zero_u"), ((48, 32, 20), "zero_d"),
                        ((64, 16, 12), "plain"), ((32, 32, 32), "plain")]:
        n = int(np.prod(shape))
        d = np.array([0.0, 0.13, 0.013, 0.05])[rng.integers(0, 4, n)]
        if kind == "zero_d":
            d = np.zeros(n)
        u0 = np.zeros(n)
        if kind != "zero_u":
            u0[rng.integers(0, n, 50)] = rng.uniform(0.2, 1.0, 50)
            u0[d == 0.0] = 0.0 if kind != "zero_d" else u0[d == 0.0]
        specs.append((shape, d, u0, 0.025 * (1 + len(specs))))
    ops = [G.assemble_diffusion(G.Grid(*sh, h=2.0), d) for sh, d, _, _ in specs]
    try:
        for op, (_, _, u0, _) in zip(ops, specs):
            op.set_state(u0)
        steps = 3
        _, infos = G.run_ensemble(ops, steps, [r for *_, r in specs], 33.5, 1e-8, metrics=False, infos=True,
                                  groups=2)
        branches = set()
        for i, (op, (shape, d, u0, rho)) in enumerate(zip(ops, specs)):
            op_o = port.stencil(shape, 2.0, d)
            u = u0
            for q in range(steps):
                inf = infos[i][q]
                branches.add(inf.branch)
                u, log = port.step(op_o, u, rho, 33.5, 1e-8, bnorm=inf.bnorm, coln=inf.coln)
                assert inf.stage_terms() == log.stage_terms(), (i, q)
            assert np.array_equal(op.get_state(), u), i
        assert {0, 2, 3} <= branches
    finally:
        for op in ops:
            op.close()


@pytest.mark.gpu
@pytest.mark.parametrize("chunks", [1, 2, 3])
def test_step_ensemble_host_bitwise_vs_oracle(port, chunks):
    """gs_step_ensemble_host: value semantics per member (u in, u' out, as the drop-in step()),
    batched in `chunks` member chunks whose copies overlap the other chunks' steps -- every
    member bitwise against the oracle given its device sums, from pinned and pageable vectors."""
    import torch
    from paper_2402_02273_b200 import gliosim as G
    shape = (48, 32, 20)
    members = _random_members(port, shape, 5, 40 + chunks)
    ops = [G.assemble_diffusion(G.Grid(*shape, h=2.0), d) for d, _, _ in members]
    try:
        ins = []
        for i, (_, u0, _) in enumerate(members):
            if i % 2 == 0:  # pinned host memory (asynchronous copies)
                t = torch.empty(u0.size, dtype=torch.float64, pin_memory=True)
                t.numpy()[:] = u0
                ins.append(t.numpy())
            else:
                ins.append(u0.copy())
        outs, infos = G.step_ensemble_host(ops, ins, [r for *_, r in members], 33.5, 1e-8, infos=True, groups=2,
                                           chunks=chunks)
        for i, (op, (d, u0, rho)) in enumerate(zip(ops, members)):
            want, log = port.step(port.stencil(shape, 2.0, d), u0, rho, 33.5, 1e-8, bnorm=infos[i].bnorm,
                                  coln=infos[i].coln)
            assert infos[i].stage_terms() == log.stage_terms(), i
            assert np.array_equal(outs[i], want), i
            assert np.array_equal(ins[i], u0), i  # inputs untouched
    finally:
        for op in ops:
            op.close()

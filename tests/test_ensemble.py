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

"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck), one process per case:

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py tma
  cases: tma (48x32x20, fused two-term TMA ring + seqsum kernels), l1 (the L1 fallback),
         cluster (32^3 single-cluster DSMEM path), ensemble (4 members, batched; group
         barriers), host (value-semantics step + ensemble host step), csr (generic CSR).
Each case runs two exponential-Euler steps with the step log (so the exact column sum runs
too) and checks the result against the oracle bit for bit."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Port  # noqa: E402
from paper_2402_02273_b200 import gliosim as G  # noqa: E402

case = sys.argv[1]
port = Port()
rng = np.random.default_rng(7)


def field(shape):
    n = int(np.prod(shape))
    d = np.array([0.0, 0.13, 0.013, 0.05])[rng.integers(0, 4, n)]
    u = np.zeros(n)
    u[rng.integers(0, n, 40)] = rng.uniform(0.2, 1.0, 40)
    u[d == 0.0] = 0.0
    return d, u


def check_run(shape, h=0.5, steps=2):
    d, u0 = field(shape)
    with G.assemble_diffusion(G.Grid(*shape, h=h), d) as op:
        op.set_state(u0)
        op.run_resident(steps, 0.025, 33.5, 1e-8, metrics=True, infos=True)
        got = op.get_state()
        path = "cluster" if op.uses_cluster() else "multi-kernel"
    op_o = port.stencil(shape, h, d)
    u = u0
    for _ in range(steps):
        u, _ = port.step(op_o, u, 0.025, 33.5, 1e-8)
    assert np.array_equal(got, u), case
    print(f"{case}: {shape} {path} ok")


if case == "tma":
    os.environ["GS_NO_CLUSTER"] = "1"
    check_run((48, 32, 20))
elif case == "l1":
    os.environ["GS_NO_CLUSTER"] = "1"
    os.environ["GS_DISABLE_TMA"] = "1"
    check_run((48, 32, 20))
elif case == "cluster":
    check_run((32, 32, 32))
elif case == "ensemble":
    shapes = [(48, 32, 20), (32, 32, 24), (64, 16, 16), (48, 32, 20)]
    ops, us, ds = [], [], []
    for s in shapes:
        d, u = field(s)
        op = G.assemble_diffusion(G.Grid(*s, h=0.5), d)
        op.set_state(u)
        ops.append(op)
        us.append(u)
        ds.append(d)
    rhos = [0.025, 0.05, 0.01, 0.1]
    G.run_ensemble(ops, 2, rhos, 33.5, 1e-8, metrics=True, infos=True, groups=2)
    for op, s, d, u, rho in zip(ops, shapes, ds, us, rhos):
        op_o = port.stencil(s, 0.5, d)
        for _ in range(2):
            u, _ = port.step(op_o, u, rho, 33.5, 1e-8)
        assert np.array_equal(op.get_state(), u)
        op.close()
    print("ensemble ok")
elif case == "host":
    s = (48, 32, 20)
    d, u = field(s)
    with G.assemble_diffusion(G.Grid(*s, h=0.5), d) as op:
        got = G.step(op, u, 0.025, 33.5, 1e-8)
        outs, _ = G.step_ensemble_host([op], [u], [0.025], 33.5, 1e-8)
    want, _ = port.step(port.stencil(s, 0.5, d), u, 0.025, 33.5, 1e-8)
    assert np.array_equal(got, want) and np.array_equal(outs[0], want)
    print("host ok")
elif case == "csr":
    n = 300
    rows = [np.sort(rng.choice(n, size=rng.integers(1, 6), replace=False)) for _ in range(n)]
    offs = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    cols = np.concatenate(rows).astype(np.int32)
    vals = rng.uniform(-1, 1, cols.size)
    b = rng.uniform(-1, 1, n)
    with G.CsrOperator(offs, cols, vals) as op:
        got = G.phi1v(2.0, op, b, 1e-10)
    want, _ = port.phi1v(2.0, port.csr(offs, cols, vals), b, 1e-10)
    assert np.array_equal(got, want)
    print("csr ok")
else:
    raise SystemExit(f"unknown case {case}")

"""Profiling driver: build a workload, run `--steps` exponential-Euler steps in one
launch, `--repeat` times (the first launch is the warm-up).  Used under ncu:

  ncu --set full -k regex:solve_kernel -s 1 -c 1 -o gpurun_out/prof python tools/prof_step.py --config C4
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import bench  # noqa: E402
from paper_2402_02273_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--repeat", type=int, default=2)
a = ap.parse_args()
w = W.get(a.config)
data, dims, labels = bench.build_case(w)
op = bench.make_operator(w, data, dims)
if labels is None:
    labels = op.labels()
u0 = bench.initial_state(w, op, labels)
for r in range(a.repeat):
    op.set_state(u0)
    t0 = time.perf_counter()
    _, inf = op.run_resident(a.steps, w.rho, w.tau, W.TOL, metrics=False, infos=True)
    dt = time.perf_counter() - t0
    print(f"launch {r}: {a.steps} steps in {dt*1e3:.2f} ms, terms {[inf[q].total_terms for q in range(a.steps)]}")
op.close()

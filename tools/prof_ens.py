"""Profiling driver for the batched ensemble (C5): build the members, run `--steps` batched
steps `--repeat` times (the first call is the warm-up).  Used under ncu:

  ncu --set full -k regex:ens_taylor -s 1 -c 1 -o gpurun_out/ens python tools/prof_ens.py
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2402_02273_b200 import ensemble as E  # noqa: E402
from paper_2402_02273_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--repeat", type=int, default=2)
ap.add_argument("--members", type=int, default=64)
a = ap.parse_args()
w = W.get("C5")
runner = E.EnsembleRunner(w, list(range(a.members)))
for r in range(a.repeat):
    runner.reset()
    t0 = time.perf_counter()
    res = runner.run(a.steps)
    print(f"call {r}: {a.steps} steps x {a.members} members in {(time.perf_counter() - t0) * 1e3:.1f} ms, "
          f"terms {sum(int(x.terms.sum()) for x in res)}")
runner.close()

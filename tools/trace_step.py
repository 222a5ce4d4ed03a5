"""Per-phase device timeline of exponential-Euler steps (grid-barrier timestamps).

  python tools/trace_step.py --config C4 --steps 2
"""
import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import bench  # noqa: E402
from paper_2402_02273_b200 import workloads as W  # noqa: E402

# a record's tag names the phase that ENDS at its timestamp
NAMES = {1: "metrics0", 2: "rhs", 3: "border", 4: "fused-first", 5: "fused-next", 6: "fixup", 7: "update",
         8: "term", 9: "branch", 10: "prep(rhs)", 11: "border", 12: "taylor-tail", 13: "update/launch", 15: "start"}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
w = W.get(a.config)
data, dims, labels = bench.build_case(w)
op = bench.make_operator(w, data, dims)
if labels is None:
    labels = op.labels()
u0 = bench.initial_state(w, op, labels)
op.set_trace(4096)
for rep in range(2):
    op.set_state(u0)
    op.run_resident(a.steps, w.rho, w.tau, W.TOL, metrics=True, infos=False)
tr = op.trace()
tot = collections.Counter()
cnt = collections.Counter()
for (tag, t), (_, tp) in zip(tr[1:], tr[:-1]):
    tot[NAMES.get(tag, tag)] += (t - tp) / 1e3
    cnt[NAMES.get(tag, tag)] += 1
span = (tr[-1][1] - tr[0][1]) / 1e3
print(f"{a.config}: {a.steps} step(s), {span:.1f} us total, {span / a.steps:.1f} us/step")
for k, v in tot.most_common():
    print(f"  {k:12s} {v:10.1f} us  {100 * v / span:5.1f}%  n={cnt[k]:4d}  {v / cnt[k]:8.2f} us each")

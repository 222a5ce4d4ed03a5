"""Steps/s of gs_run (kernel timing off) per workload under two environments, back to back:
the A/B tool for build-time-free switches (GS_TREE_SUMS, GS_NO_GRAPH, GS_LOCK_C0, ...).

  python tools/env_ab.py "GS_TREE_SUMS=1" C1 C2 C3 C4
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, time, json
sys.path.insert(0, %r)
import bench
from paper_2402_02273_b200 import workloads as W
w = W.get(%r)
data, dims, labels = bench.build_case(w)
op = bench.make_operator(w, data, dims)
if labels is None: labels = op.labels()
u0 = bench.initial_state(w, op, labels)
steps = 200 if w.n <= 2**21 else 10
best = 1e9
for rep in range(4):
    op.set_state(u0)
    t = time.perf_counter()
    op.run_resident(steps, w.rho, w.tau, W.TOL, metrics=True, infos=False)
    best = min(best, time.perf_counter() - t)
print(json.dumps({"steps_per_s": steps / best, "steps": steps}))
'''
env_b = dict(kv.split("=", 1) for kv in sys.argv[1].split(",") if kv)
for cfg in sys.argv[2:]:
    for mode, env in (("A", {}), ("B " + sys.argv[1], env_b), ("A", {})):
        out = subprocess.run([sys.executable, "-c", CODE % (ROOT, cfg)], capture_output=True, text=True,
                             env={**os.environ, **env})
        try:
            r = json.loads(out.stdout.strip().splitlines()[-1])
            print(cfg, mode, round(r["steps_per_s"], 1), flush=True)
        except Exception:
            print(cfg, mode, "failed", out.stderr[-400:], flush=True)

"""CUDA-graph replay vs direct launches for gs_run (kernel timing off), per workload.

  python tools/graph_ab.py C1 C2 C4
"""
import os
import subprocess
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, time, json
sys.path.insert(0, %r)
import bench
import numpy as np
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
for cfg in sys.argv[1:]:
    for mode, env in (("graph", {}), ("direct", {"GS_NO_GRAPH": "1"})):
        out = subprocess.run([sys.executable, "-c", CODE % (ROOT, cfg)], capture_output=True, text=True,
                             env={**os.environ, **env})
        try:
            r = json.loads(out.stdout.strip().splitlines()[-1])
            print(cfg, mode, round(r["steps_per_s"], 1))
        except Exception:
            print(cfg, mode, "failed", out.stderr[-400:])

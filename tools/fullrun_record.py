"""Full-run parity record at a BASELINE config (default: C4, all 100 steps) against the
compiled reference's run() -- the long form of tests/test_gpu_fullrun.py (minutes of reference
time on the host cores).  Writes a JSON record:

  python tools/fullrun_record.py --config C4 --steps 100 --out profiles/r02_c4_trajectory_parity.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import bench  # noqa: E402
import fullrun as FR  # noqa: E402
from oracle import Port, Ref  # noqa: E402
from paper_2402_02273_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--out", required=True)
a = ap.parse_args()
w = W.get(a.config)
data, dims, labels = bench.build_case(w)
op = bench.make_operator(w, data, dims)
ref, port = Ref(), Port()
tic = time.perf_counter()
want = ref.resample(data, dims[0], dims[1], dims[2], (w.nx, w.ny, w.nz))
labels = op.labels()
rec = dict(tool="tools/fullrun_record.py", host_cores=FR.host_cores(),
           material_map_equal=labels.tobytes() == want.tobytes(),
           path=("single-cluster" if op.uses_cluster() else
                 "resident tiles (2-D)" if op.uses_flat2d() else "multi-kernel"))
u0 = bench.initial_state(w, op, labels)
center = W.seed_points(w, labels)[0]
FR.full_run_parity(a.config, op, labels, u0, a.steps, w.rho, w.tau, W.TOL, center, port, ref, record=rec,
                   log=lambda m: print(m, flush=True))
rec["wall_seconds"] = time.perf_counter() - tic
try:
    FR.assert_record(rec)
    rec["gates_pass"] = True
except AssertionError as e:
    rec["gates_pass"] = False
    rec["gate_failure"] = str(e)
os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
with open(a.out, "w") as f:
    json.dump(rec, f, indent=1, default=str)
print(json.dumps({k: v for k, v in rec.items() if k not in ("per_step", "terms_per_step")}, default=str))

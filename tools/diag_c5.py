"""Diagnose the batched ensemble on a few C5 members: NaN / divergence per step against
per-member gs_run (one-off debugging aid)."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_02273_b200 import ensemble as E, gliosim as G, workloads as W, phantom

w = W.get("C5")
rhos = [W.member_rho(w, mb) for mb in range(w.members)]
pick = [int(np.argmin(rhos)), w.members // 2, int(np.argmax(rhos))]
rnd = int(phantom.uniform01(w.seed, 77, 1)[0] * w.members)
while rnd in pick:
    rnd = (rnd + 1) % w.members
pick.append(rnd)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
print("pick", pick, [rhos[p] for p in pick], flush=True)
runner = E.EnsembleRunner(w, pick)
seq = E.EnsembleRunner(w, pick)
runner.reset(); seq.reset()
for k in range(steps):
    _, inf = G.run_ensemble(runner.ops, 1, runner.rhos, w.tau, W.TOL, metrics=False, infos=True)
    line = []
    for i, (op, op2) in enumerate(zip(runner.ops, seq.ops)):
        _, inf2 = op2.run_resident(1, seq.rhos[i], w.tau, W.TOL, metrics=False, infos=True)
        a, b = op.get_state(), op2.get_state()
        nan = int(np.isnan(a).sum())
        rel = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
        line.append(f"m{pick[i]}: nan={nan} rel={rel:.1e} t={inf[i][0].total_terms}/{inf2[0].total_terms} s={inf[i][0].s}/{inf2[0].s} br={inf[i][0].branch} g={inf[i][0].gamma:.3e}")
    print(k + 1, " | ".join(line), flush=True)

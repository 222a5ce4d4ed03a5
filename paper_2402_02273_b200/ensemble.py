"""C5: an ensemble of independent runs (parameter sweep / supermodeling), replicas only.

Members share nothing -- different phantoms, seed points and rho -- so the multi-GPU plan
is a static partition of members over ranks (one process per GPU) with no data-path
collective; the only communication is gathering each member's per-step metrics to rank 0
at the end (torch.distributed, NCCL on GPUs or gloo on CPU).  SURVEY.md 8(e).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import workloads as W


def members_for_rank(n_members: int, rank: int, world: int) -> list[int]:
    """Contiguous balanced blocks: rank r gets members [r*n/W, (r+1)*n/W)."""
    lo = rank * n_members // world
    hi = (rank + 1) * n_members // world
    return list(range(lo, hi))


@dataclass
class MemberResult:
    member: int
    rho: float
    steps: int
    metrics: np.ndarray      # (steps+1, 4): total_mass, max, min, radius
    terms: np.ndarray        # Taylor terms per step
    checksum: float          # sum of the final state (sanity)
    stage_terms: list | None = None  # per step, the Taylor terms of each stage (the step log)


class EnsembleRunner:
    """Holds one resident operator + state per member of this rank (inputs stay in HBM)."""

    def __init__(self, w: W.Workload, members: list[int], device: int = 0):
        from . import gliosim as G
        self.G = G
        self.w = w
        self.members = members
        self.ops, self.u0, self.centers, self.rhos = [], [], [], []
        cfg = G.SimConfig(d_white=W.D_WHITE, d_gray=W.D_GRAY)
        for mb in members:
            data, wd, ht, sl = W.intensity(w, mb)
            op = G.StencilOperator.from_intensity(G.Grid(w.nx, w.ny, w.nz, w.h), data, wd, ht, sl, cfg, device=device)
            labels = op.labels()
            u = None
            centers = W.seed_points(w, labels, mb)
            for c in centers:
                sc = G.SimConfig(seed_center=c, seed_amplitude=1.0, seed_width=W.seed_width(w))
                ui = G.seed_initial(op, sc, mask=True)
                u = ui if u is None else np.maximum(u, ui)
            self.ops.append(op)
            self.u0.append(u)
            self.centers.append(centers[0])
            self.rhos.append(W.member_rho(w, mb))

    def reset(self):
        for op, u in zip(self.ops, self.u0):
            op.set_state(u)

    def run(self, steps: int, batched: bool = True, groups: int = 0) -> list[MemberResult]:
        """Advance every member `steps` steps.  batched: one gs_run_ensemble call (the step's
        kernels serve all members; the Taylor launch runs `groups` members at a time on
        groups of SMs); otherwise one gs_run per member, each on the whole GPU."""
        if batched and self.members:
            m, inf = self.G.run_ensemble(self.ops, steps, self.rhos, self.w.tau, W.TOL, np.zeros((len(self.ops), 3)),
                                         np.array(self.centers, dtype=np.float64), 0.1, metrics=True, infos=True,
                                         groups=groups)
            out = []
            for i, (mb, rho) in enumerate(zip(self.members, self.rhos)):
                met = np.array([[x.total_mass, x.max_density, x.min_density, x.radius] for x in m[i]])
                terms = np.array([inf[i][q].total_terms for q in range(steps)])
                st = [inf[i][q].stage_terms() for q in range(steps)]
                out.append(MemberResult(mb, rho, steps, met, terms, float("nan"), st))
            return out
        out = []
        for mb, op, c, rho in zip(self.members, self.ops, self.centers, self.rhos):
            m, inf = op.run_resident(steps, rho, self.w.tau, W.TOL, (0.0, 0.0, 0.0), c, 0.1, metrics=True, infos=True)
            met = np.array([[x.total_mass, x.max_density, x.min_density, x.radius] for x in m])
            terms = np.array([inf[q].total_terms for q in range(steps)])
            out.append(MemberResult(mb, rho, steps, met, terms, float("nan"), [inf[q].stage_terms() for q in range(steps)]))
        return out

    def close(self):
        for op in self.ops:
            op.close()


def gather_results(results: list[MemberResult], n_members: int, steps: int, dist=None):
    """Gather every member's metrics to rank 0 as an (n_members, steps+1, 4) array (NaN where
    a member is missing).  With `dist` (torch.distributed) uses all_gather_object."""
    table = np.full((n_members, steps + 1, 4), np.nan)
    terms = np.zeros((n_members, steps), dtype=np.int64)
    for r in results:
        table[r.member] = r.metrics
        terms[r.member] = r.terms
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return table, terms
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, [(r.member, r.metrics, r.terms) for r in results])
    for part in parts:
        for mb, met, tm in part:
            table[mb] = met
            terms[mb] = tm
    return table, terms

"""Full-run parity harness -- TEST INFRASTRUCTURE (imports oracle/).

North_star's gates on BASELINE.json's configurations, checked against the reference's own
time loop `gliosim::run` (/root/reference/proj/src/integrator.cpp:91-138):

* material map: the device labels `memcmp`-equal the reference's `resample`
  (imaging.cpp:125-141) of the same input bytes;
* per step (one-step mode): the GPU's state u_n is fed to the C restatement of `step`
  (oracle/gliosim_oracle.c, pinned bitwise to the reference); the oracle's (s, m) and
  terms per stage must EQUAL the GPU's, and its u_{n+1} must be within relative L2 1e-10
  of the GPU's;
* full run (trajectory mode): the GPU's production loop (`gs_run`, one call for every
  step) against the compiled, unmodified reference's `run()` started from the same u0:
  final u within relative L2 1e-8, and every node's metrics (compute_metrics,
  integrator.cpp:65-89) close;
* determinism: the state after the stepwise pass (one `gs_run` call per step, direct
  launches) equals the production pass (one call, graph replay) bit for bit.

The oracle calls release the GIL (ctypes), so the one-step checks run on a thread pool
over the host cores while the GPU produces the next states.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import time

import numpy as np

PER_STEP_TOL = 1e-10
FULL_RUN_TOL = 1e-8


def rel_l2(a, b):
    """Relative L2 distance; NaN-aware: a NaN in one vector and not at the same place in the
    other is infinitely far, NaNs in both at the same places are equal (a run that overflowed,
    as the reference's explicit logistic term does for rho tau > 3, ends in NaN in both)."""
    a = np.asarray(a)
    b = np.asarray(b)
    na, nb_ = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb_):
        return float("inf")
    if na.any():
        a, b = a[~na], b[~na]
    fin = np.isfinite(a) & np.isfinite(b)
    if not np.array_equal(a[~fin], b[~fin]):
        return float("inf")
    a, b = a[fin], b[fin]
    nb = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b) / nb) if nb else float(np.linalg.norm(a - b))


def bitwise(a, b):
    """Equal bit for bit, any NaN equal to any NaN (payloads differ between x86 and the GPU)."""
    return bool(np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True))


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _info_tuple(inf):
    return (int(inf.s), int(inf.m), tuple(inf.stage_terms()))


def _log_tuple(log):
    return (int(log.s), int(log.m), tuple(log.stage_terms()))


def check_one_step_sequence(port, op_o, states, rho, tau, tol, threads=None, record=None):
    """states: iterable of (k, gpu_info_k, u_k, u_{k+1}) -- the GPU's input and output of
    step k+1 -- or of (k, info, u_k, u_{k+1}, op_o, rho) when members differ.  Each is
    checked on a thread pool against the oracle's step(u_k).  Returns the list of per-step
    dicts (rel_l2, equal decision log), ordered by k."""
    threads = threads or host_cores()
    out = {}

    def one(k, info_t, u_in, u_out, op_k, rho_k):
        want, log = port.step(op_k, u_in, rho_k, tau, tol)
        return k, info_t, _log_tuple(log), rel_l2(u_out, want), int(log.total_terms), bitwise(u_out, want)

    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        pend = set()
        for item in states:
            k, inf, u_in, u_out = item[:4]
            op_k, rho_k = (item[4], item[5]) if len(item) > 4 else (op_o, rho)
            pend.add(ex.submit(one, k, _info_tuple(inf), u_in, u_out, op_k, rho_k))
            # bound the states held in memory (128 MiB each at 256^3)
            while len(pend) >= 2 * threads:
                done, pend = cf.wait(pend, return_when=cf.FIRST_COMPLETED)
                for f in done:
                    k2, it, lt, r, tt, bw = f.result()
                    out[k2] = dict(key=k2, step=(k2[-1] if isinstance(k2, tuple) else k2) + 1, gpu=it, oracle=lt,
                                   rel_l2=r, terms=tt, bitwise=bw)
        for f in cf.as_completed(pend):
            k2, it, lt, r, tt, bw = f.result()
            out[k2] = dict(key=k2, step=(k2[-1] if isinstance(k2, tuple) else k2) + 1, gpu=it, oracle=lt,
                           rel_l2=r, terms=tt, bitwise=bw)
    rows = [out[k] for k in sorted(out)]
    if record is not None:
        record["per_step"] = [dict(step=r["step"], key=r["key"], s=r["gpu"][0], m=r["gpu"][1], terms=list(r["gpu"][2]),
                                   decisions_equal=r["gpu"] == r["oracle"], rel_l2=r["rel_l2"], bitwise=r["bitwise"])
                              for r in rows]
    return rows


def stepwise_states(op, u0, n_steps, rho, tau, tol):
    """The GPU trajectory one gs_run call per step: yields (k, info_k, u_k, u_{k+1})."""
    op.set_state(u0)
    u = np.array(u0, dtype=np.float64, copy=True)
    for k in range(n_steps):
        _, inf = op.run_resident(1, rho, tau, tol, metrics=False, infos=True)
        nxt = op.get_state()
        yield k, inf[0], u, nxt
        u = nxt


def production_run(op, u0, n_steps, rho, tau, tol, center):
    """The GPU's production loop: ONE gs_run call for every step (graph replay), metrics at
    every node, step infos."""
    op.set_state(u0)
    m, inf = op.run_resident(n_steps, rho, tau, tol, (0.0, 0.0, 0.0), center, 0.1, metrics=True, infos=True)
    met = np.array([[x.total_mass, x.max_density, x.min_density, x.radius] for x in m])
    return op.get_state(), met, [_info_tuple(x) for x in inf[:n_steps]]


def compare_metrics(got, want):
    """Per-node metric differences: mass/max/min relative to max(|u0| mass, 1e-300); radius
    exact lattice values compared relatively."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    same = (got == want) | (np.isnan(got) & np.isnan(want))
    scale = np.maximum(np.abs(want), 1e-300)
    with np.errstate(invalid="ignore", over="ignore"):
        diff = np.where(same, 0.0, np.abs(got - want) / scale)
    diff = np.where(np.isnan(diff), np.inf, diff)
    return float(np.max(diff)) if diff.size else 0.0


def full_run_parity(name, op, labels, u0, n_steps, rho, tau, tol, center, port, ref, t0=150.0,
                    threads=None, per_step=True, record=None, log=print):
    """All gates for one run.  Returns a JSON-able record; asserts nothing itself (the
    caller asserts on the record so a tool can save a failing record too)."""
    rec = dict(config=name, steps=n_steps, rho=rho, tau=tau, tol=tol, voxels=int(u0.size))
    if record is not None:
        record.update(rec)
        rec = record
    shape = op.grid.shape
    h = op.grid.h
    d = port.diffusion_from_labels(labels)
    op_o = port.stencil(shape, h, d)
    tic = time.perf_counter()
    if per_step:
        rows = check_one_step_sequence(port, op_o, stepwise_states(op, u0, n_steps, rho, tau, tol), rho, tau, tol,
                                       threads=threads, record=rec)
        stepwise_final = op.get_state()
        rec["per_step_max_rel_l2"] = max(r["rel_l2"] for r in rows)
        rec["per_step_decisions_equal"] = all(r["gpu"] == r["oracle"] for r in rows)
        rec["per_step_bitwise"] = all(r["bitwise"] for r in rows)
        rec["per_step_seconds"] = time.perf_counter() - tic
        log(f"[{name}] one-step mode: {n_steps} steps, max rel L2 {rec['per_step_max_rel_l2']:.3e}, "
            f"decisions equal {rec['per_step_decisions_equal']}, bitwise {rec['per_step_bitwise']} "
            f"({rec['per_step_seconds']:.1f} s)")
    u_gpu, met_gpu, infos = production_run(op, u0, n_steps, rho, tau, tol, center)
    if per_step:
        rec["stepwise_equals_production_bitwise"] = bitwise(stepwise_final, u_gpu)
        rec["production_decisions_equal_stepwise"] = [tuple(r["gpu"]) for r in rows] == infos
    rec["terms_per_step"] = [int(sum(t[2])) for t in infos]
    # the reference's own run(): t_end chosen so TimeGrid::tau() == tau exactly
    t_end = t0 + n_steps * tau
    assert (t_end - t0) / n_steps == tau
    tic = time.perf_counter()
    cores = threads or host_cores()
    u_ref, met_ref, secs = ref.run(shape, h, d, u0, n_steps, rho, t0, t_end, tol, center, 0.1, workers=cores)
    rec["reference_run_seconds"] = time.perf_counter() - tic
    rec["reference_step_seconds"] = secs
    rec["reference_workers"] = cores
    rec["final_rel_l2_vs_reference"] = rel_l2(u_gpu, u_ref)
    rec["final_bitwise_vs_reference"] = bitwise(u_gpu, u_ref)
    rec["metrics_bitwise_nodes"] = int(sum(bitwise(a, b) for a, b in zip(met_gpu, met_ref)))
    rec["metrics_max_rel_diff"] = compare_metrics(met_gpu, met_ref)
    rec["metrics_mass_max_rel_diff"] = compare_metrics(met_gpu[:, 0], met_ref[:, 0])
    rec["radius_equal_nodes"] = int(np.sum(met_gpu[:, 3] == met_ref[:, 3]))
    rec["nodes"] = int(met_ref.shape[0])
    log(f"[{name}] trajectory: final rel L2 vs reference run() {rec['final_rel_l2_vs_reference']:.3e} "
        f"(bitwise {rec['final_bitwise_vs_reference']}), "
        f"metrics max rel diff {rec['metrics_max_rel_diff']:.3e}, radius equal at "
        f"{rec['radius_equal_nodes']}/{rec['nodes']} nodes (reference {rec['reference_run_seconds']:.1f} s "
        f"on {cores} workers)")
    return rec


def assert_record(rec, per_step=True, exact=True):
    """The gates; exact: also bit-for-bit (the device sums are the reference's sequential ones,
    so every step and the whole trajectory are the reference's bits)."""
    if per_step:
        bad = [r for r in rec["per_step"] if not r["decisions_equal"]]
        assert not bad, f"{rec['config']}: (s, m, terms) differ at steps {[r['step'] for r in bad][:10]}"
        assert rec["per_step_max_rel_l2"] <= PER_STEP_TOL, rec["per_step_max_rel_l2"]
        assert rec["stepwise_equals_production_bitwise"], "stepwise and production GPU runs differ"
        if exact:
            assert rec["per_step_bitwise"], [r["step"] for r in rec["per_step"] if not r["bitwise"]][:10]
        assert rec["production_decisions_equal_stepwise"]
    assert rec["final_rel_l2_vs_reference"] <= FULL_RUN_TOL, rec["final_rel_l2_vs_reference"]
    if exact:
        assert rec["final_bitwise_vs_reference"], "final state not bit-identical to the reference's run()"
    assert rec["metrics_mass_max_rel_diff"] <= 1e-8, rec["metrics_mass_max_rel_diff"]

"""bench.py -- exponential-Euler throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

One "step" = one exponential-Euler step (integrator.cpp:52-63) of the configured
workload (default C4: 256^3 fp64 shell phantom, the headline config).  Our arm runs the
CUDA path with all state resident in HBM; the reported ``value`` is whole-job steps/s
(N independent replicas under torchrun: the path does not shard, DESIGN.md "replicas
only").  ``e2e`` is the same metric through the drop-in step() call with host buffers
(pinned H2D of u, the step, D2H of the new u every step).  ``roofline`` covers the
persistent solve kernel (the only kernel in the timed region) against the measured HBM
copy peak; ``cpu_baseline`` is the UNMODIFIED reference (oracle/_ref) timed on this
host on full-grid steps of the same workload (one step with all host cores, one with one).
``--impl reference`` times that reference alone: full-grid gliosim::run steps on all host
cores, as many of the requested steps as fit in --ref-budget seconds.

Working set at C4: u, b, f x2, T x2 = 6 x 128 MiB fp64 (+ 16 MiB labels) >> 126 MB L2,
so no L2 flush is needed between steps ("inputs larger than L2").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_TERM = 33   # per voxel per Taylor term: T 8 + f 8 + label 1 read, T 8 + f 8 write
BYTES_PER_STEP = 49   # per voxel per step outside the terms: RHS 17, bordered column 8, update 24
# Fused two-term sweep: one HBM pass per TWO Taylor terms.
BYTES_PER_SWEEP = 33  # read X 8 + (F or b/gamma) 8 + label 1, write T2 8 + F1 8
BYTES_FIRST_ZERO = 25  # stage-0 first sweep: read b/gamma 8 + label 1, write 16
BYTES_IMPLICIT = 8    # a stage starting from an implicit f = F + T reads T as well (summed in smem)


def taylor_bytes_per_voxel(info):
    """Algorithmic bytes per voxel of one taylor_kernel launch (one step), from its term log.

    A stage that ended on an even term count leaves f = F1 + T2 implicit; the next stage's
    first sweep reads both.  Exact-maxima reruns (info.reruns) are not algorithmic bytes:
    they are counted in the launch time only."""
    terms = info if isinstance(info, (list, tuple)) else info.stage_terms()
    sweeps = sum((t + 1) // 2 for t in terms)
    implicit = sum(1 for k in range(1, len(terms)) if terms[k - 1] % 2 == 0)
    return BYTES_FIRST_ZERO + BYTES_PER_SWEEP * (sweeps - 1) + BYTES_IMPLICIT * implicit, sweeps, implicit


def timed_launches(op, steps, graph_pass):
    """Kernels of this library launched inside the timed region (gs_capi.cu launch_solve): the
    single-cluster path is one launch per call; otherwise one metrics launch, then per step prep,
    border, Taylor, update, the tile and item pass of each of the two exact sums (seqsum) and,
    in the graph-replayed production pass, the one-thread step counter."""
    if op.uses_cluster():
        return 1
    per_step = 4 + (0 if os.environ.get("GS_TREE_SUMS") else 4)
    if graph_pass and steps >= 2 and not os.environ.get("GS_NO_GRAPH"):
        per_step += 1
    return steps * per_step + 1


def l2_note(n):
    ws = 7 * 8 * n / 2 ** 20
    if ws > 126:
        return f"working set 7 x {8 * n / 2 ** 20:.0f} MiB fp64 = {ws:.0f} MiB > 126 MB L2 (no flush needed)"
    return (f"working set {ws:.1f} MiB fits the 126 MB L2: the steps of one run follow each other on the same "
            "vectors, so a run's steady state IS L2-resident; not flushed between steps (that would time a cold "
            "start no run has); the roofline fraction against HBM is not meaningful here (SURVEY 8d)")


FLAT2D_K = 4  # Taylor terms per round of the resident-tile 2-D kernel (gs_flat2d.cuh, k2dK)


def flat2d_bytes_per_voxel(info):
    """The 2-D resident-tile kernel (taylor2d_kernel): per round (K = 4 terms, one grid barrier)
    a CTA writes its tile's f after each level and T_K (5 x 8 B per voxel) and reloads one 40 x 40
    box (12.5 B per tile voxel); the state itself never leaves the SM.  Returns
    (bytes per voxel, rounds, 0)."""
    terms = info if isinstance(info, (list, tuple)) else info.stage_terms()
    rounds = sum((t + FLAT2D_K - 1) // FLAT2D_K for t in terms)
    return rounds * (8 * (FLAT2D_K + 1) + 8 * 1600 / 1024), rounds, 0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 10 at 256^3 and for the reference arm; the workload's own run "
                         "length for C1/C2/C3/C5, whose per-call set-up -- graph capture, staging -- would "
                         "otherwise weigh on a few sub-millisecond steps)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=30.0,
                    help="CPU time budget of the cpu_baseline sample (at least one full-grid reference step)")
    ap.add_argument("--ref-budget", type=float, default=600.0,
                    help="--impl reference: timed seconds after which no further full-grid step starts")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def under_launcher() -> bool:
    """torchrun (torch.distributed.run) sets these: use the process group even at world 1."""
    return all(k in os.environ for k in ("RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"))


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region: an NVML
    thread polls every 10 ms between __enter__ and __exit__, with one sample on entry and one
    on exit, so even a short region has samples; nvidia-smi -lms is the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.max_mhz = 0.0
        self.nvml = None
        self.proc = None
        self.path = f"/tmp/gs_clocks_{os.getpid()}.csv"
        # 10 ms: NVML queries from a second thread cost launch-bound runs (C1) ~3% at 2 ms
        self.period = float(os.environ.get("GS_CLOCKS_PERIOD_MS", "10")) / 1e3
        try:
            if os.environ.get("GS_CLOCKS") == "smi":
                raise RuntimeError("nvidia-smi sampling requested")
            import threading

            import pynvml
            import torch
            pynvml.nvmlInit()
            nvml_index = torch.cuda._get_nvml_device_index(index)  # honours CUDA_VISIBLE_DEVICES
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(nvml_index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
            self.nvml = pynvml
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
        except Exception:
            self.nvml = None

    def _sample(self):
        N = self.nvml
        sm = float(N.nvmlDeviceGetClockInfo(self.handle, N.NVML_CLOCK_SM))
        bits = N.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
        self.samples.append((sm, {nm for nm, attr in self.REASONS if bits & getattr(N, attr)}))

    def _poll(self):
        while not self.stop.wait(self.period):
            try:
                self._sample()
            except Exception:
                return

    def __enter__(self):
        if self.nvml:
            self._sample()
            self.thread.start()
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.thread.join(timeout=5)
            try:
                self._sample()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.nvml:
            if not self.samples:
                return None
            reasons = set().union(*(r for _, r in self.samples))
            return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(reasons), "samples": len(self.samples),
                    "source": f"nvml every {self.period * 1e3:g} ms (+ entry/exit samples)"}
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            return None
        sm, mx, reasons = [], 0.0, set()
        names = [nm for nm, _ in self.REASONS]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for nm, val in zip(names, r[4:8]):
                    if val.strip() == "Active":
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvidia-smi -lms 50"}


def build_case(w, member=0):
    """Host inputs for a workload: intensity bytes, labels (for the CPU side), u0 pieces."""
    from paper_2402_02273_b200 import workloads as W
    data, wd, ht, sl = W.intensity(w, member)
    table = W.classify_table()
    if w.stack_slices:
        from paper_2402_02273_b200 import phantom  # noqa: F401
        # labels come from the device resample; the CPU side gets them back from the GPU
        labels = None
    else:
        labels = table[data]
    return data, (wd, ht, sl), labels


def make_operator(w, data, dims):
    from paper_2402_02273_b200 import gliosim as G
    from paper_2402_02273_b200 import workloads as W
    cfg = G.SimConfig(d_white=W.D_WHITE, d_gray=W.D_GRAY)
    return G.StencilOperator.from_intensity(G.Grid(w.nx, w.ny, w.nz, w.h), data, dims[0], dims[1], dims[2], cfg)


def initial_state(w, op, labels):
    from paper_2402_02273_b200 import gliosim as G
    from paper_2402_02273_b200 import workloads as W
    u = None
    for c in W.seed_points(w, labels):
        cfg = G.SimConfig(seed_center=c, seed_amplitude=1.0, seed_width=W.seed_width(w))
        ui = G.seed_initial(op, cfg, mask=True)
        u = ui if u is None else np.maximum(u, ui)
    return u


# ------------------------------------------------------------------------------------------
# CPU side: the unmodified reference on the full grid of the workload
# ------------------------------------------------------------------------------------------

def cpu_reference_sample(w, labels, u0, steps, warmup=0, rho=None, cores=None, budget_s=None):
    """Time the reference's own run() loop (RunTimings::step_seconds, integrator.cpp:123-125)
    on the FULL grid of the workload with workers = all host cores (or `cores`): `warmup`
    untimed steps, then `steps` timed steps, one run() call per step so every step is its own
    sample (the operator assembly of each call is outside step_seconds).  budget_s caps the
    timed steps when the first one shows they would not fit.  The C port stands in only where
    oracle/_ref is absent."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Port
    try:
        from oracle import Ref
        ref = Ref()
        kind = "reference"
    except Exception:
        ref = None
        kind = "port"
    from paper_2402_02273_b200 import workloads as W
    cores = cores or host_cores()
    shape = (w.nx, w.ny, w.nz)
    d = np.array([0.0, W.D_WHITE, W.D_GRAY, 0.0])[labels]
    center = (0.0, 0.0, 0.0)
    port = Port()
    op_p = port.stencil(shape, w.h, d)
    rho = w.rho if rho is None else rho

    def one(u):
        if ref:
            u2, _, secs = ref.run(shape, w.h, d, u, 1, rho, W.T0, W.T0 + W.TAU, W.TOL, center, workers=cores)
            return u2, secs
        t0 = time.perf_counter()
        u2, _, _ = port.run(op_p, u, 1, rho, W.TAU, W.TOL, center)
        return u2, time.perf_counter() - t0

    u = u0
    for _ in range(warmup):
        u, _ = one(u)
    times = []
    for k in range(max(1, steps)):
        u, secs = one(u)
        times.append(secs)
        if budget_s is not None and k == 0:
            steps = max(1, min(steps, int(budget_s / max(secs, 1e-9))))
        if len(times) >= steps:
            break
    return {"kind": kind, "cores": cores if kind == "reference" else 1, "shape": shape, "step_times": times,
            "steps": len(times), "warmup": warmup}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------------------------------------
# arms
# ------------------------------------------------------------------------------------------

def run_ours(args, w, rank, world, local):
    import torch
    from paper_2402_02273_b200 import gliosim as G
    from paper_2402_02273_b200 import workloads as W

    torch.cuda.set_device(local)
    dist = None
    if world > 1 or under_launcher():
        import torch.distributed as D
        D.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = D

    data, dims, labels = build_case(w)
    op = make_operator(w, data, dims)
    if labels is None:
        labels = op.labels()
    u0 = initial_state(w, op, labels)
    stream = torch.cuda.ExternalStream(op.stream_handle())
    peak, peak_kind = measured_peak()

    # warm-up (untimed): W steps
    op.set_state(u0)
    op.run_resident(args.warmup, w.rho, w.tau, W.TOL, metrics=False, infos=False)
    op.set_state(u0)
    torch.cuda.synchronize()

    # timed: exactly K steps (one gs_run call = the launch sequence prep/border/taylor/update per
    # step), device-timed with CUDA events on the launching stream.  At 256^3 (10 ms steps) the
    # per-kernel events and the step log sit inside the timed region.  On the small grids (steps
    # of 0.06-0.7 ms: C1-C3) per-kernel events force direct launches instead of the production
    # path's graph replay and the step log forces the exact bordered column sum every step, which
    # together cost 10-25% there: `value` is then the production path (metrics at every node, no
    # events between kernels, no step log), and a second pass of the same K steps from the same
    # u0, inside bench.py, takes the per-kernel events and the step log for the roofline.
    separate = w.n <= 128 ** 3 and not os.environ.get("GS_BENCH_ONE_PASS")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    if not separate:
        op.set_kernel_timing(True)
    with Clocks(local) as clk:
        ev0.record(stream)
        metrics, infos = op.run_resident(args.steps, w.rho, w.tau, W.TOL, (0, 0, 0), (0, 0, 0), 0.1,
                                         metrics=True, infos=not separate)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    pass2_ms = None
    if separate:
        op.set_state(u0)
        op.set_kernel_timing(True)
        torch.cuda.synchronize()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        _, infos = op.run_resident(args.steps, w.rho, w.tau, W.TOL, (0, 0, 0), (0, 0, 0), 0.1,
                                   metrics=True, infos=True)
        p1.record(stream)
        torch.cuda.synchronize()
        pass2_ms = p0.elapsed_time(p1)
    ktimes = op.kernel_times()
    op.set_kernel_timing(False)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    terms = [infos[q].total_terms for q in range(args.steps)]
    sm = [(infos[q].s, infos[q].m) for q in range(args.steps)]
    ms_step = ms / args.steps
    value = world * args.steps / (ms / 1e3)
    # roofline of the dominant kernel (taylor_kernel): algorithmic bytes of the fused design
    flat2d = op.uses_flat2d() and not op.uses_cluster()
    tb = [(flat2d_bytes_per_voxel(infos[q]) if flat2d else taylor_bytes_per_voxel(infos[q])) for q in range(args.steps)]
    taylor_ms, taylor_n = ktimes["taylor"]
    taylor_bytes = w.n * sum(b for b, _, _ in tb)
    achieved = taylor_bytes / (taylor_ms / 1e3) / 1e9
    single_term_equiv = w.n * BYTES_PER_TERM * sum(terms) / (taylor_ms / 1e3) / 1e9
    step_bytes = taylor_bytes + w.n * BYTES_PER_STEP * args.steps

    # e2e through the drop-in step() with host buffers (pinned H2D + step + D2H)
    e2e = None
    if not args.no_e2e:
        import ctypes as C
        from paper_2402_02273_b200 import _native as N
        pin_in = torch.empty(w.n, dtype=torch.float64, pin_memory=True)
        pin_out = torch.empty(w.n, dtype=torch.float64, pin_memory=True)
        pin_in.numpy()[:] = u0
        lib = op.lib
        info = N.GsStepInfo()
        k_e2e = max(1, min(args.steps, 5))
        for _ in range(1):
            rc = lib.gs_step_host(op.ctx, pin_in.numpy(), w.rho, w.tau, W.TOL, pin_out.numpy(), C.byref(info))
            assert rc == 0
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        # device-timed on the context's stream: the events bracket the first H2D and the
        # last D2H (gs_step_host is synchronous, so host gaps between calls are included)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        src, dst = pin_in, pin_out
        for _ in range(k_e2e):
            rc = lib.gs_step_host(op.ctx, src.numpy(), w.rho, w.tau, W.TOL, dst.numpy(), C.byref(info))
            assert rc == 0
            src, dst = dst, src
        e1.record(stream)
        torch.cuda.synchronize()
        dt = e0.elapsed_time(e1) / 1e3
        if dist:
            t = torch.tensor([dt], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": world * k_e2e / dt, "unit": "steps/s", "h2d_bytes_per_step": 8 * w.n,
               "d2h_bytes_per_step": 8 * w.n, "api": "gs_step_host (drop-in step(): u H2D from pinned, u' D2H)",
               "steps": k_e2e}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            # one full-grid step of the reference on all host cores (~15 s at 256^3 on 16 cores),
            # then one with workers = 1; no extrapolation
            sample = cpu_reference_sample(w, labels, u0, 1, budget_s=args.cpu_seconds)
            t = float(np.mean(sample["step_times"]))
            cpu = {"value": 1.0 / t, "unit": "steps/s", "cores": sample["cores"], "kind": sample["kind"],
                   "sample": (f"{sample['steps']} gliosim::run step(s) of the full {w.nx}x{w.ny}x{w.nz} grid from the "
                              f"same u0 (workers={sample['cores']}), {t:.2f} s/step (RunTimings::step_seconds)")}
            if sample["kind"] == "reference" and sample["cores"] > 1:
                one = cpu_reference_sample(w, labels, u0, 1, cores=1)
                t1 = float(one["step_times"][0])
                cpu.update({"value_1core": 1.0 / t1,
                            "sample_1core": f"1 gliosim::run step of the full grid with workers=1, {t1:.2f} s"})
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "steps/s", "cores": host_cores(), "kind": "unavailable",
                   "sample": f"failed: {e}"}

    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(w.name)
            if tr:
                # dram bytes of one taylor_kernel launch from the committed ncu capture
                traffic = tr["taylor_dram_bytes_per_launch"]
    except Exception:
        pass

    line = {
        "metric": "expEuler steps/s at 256^3 fp64" if w.name.startswith("C4") else f"expEuler steps/s ({w.name})",
        "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded shell phantom, BASELINE.json config)",
        "config": {"workload": f"{w.name}: {w.note}", "grid": [w.nx, w.ny, w.nz], "h_mm": w.h, "rho": w.rho,
                   "tau_days": w.tau, "tol": W.TOL, "sigma_vox": w.sigma_vox,
                   "parallelism": f"replicas x{world} (path does not shard)",
                   "l2": l2_note(w.n),
                   "s_m": sorted(set(sm)), "terms_per_step": float(np.mean(terms))},
        "taylor_terms_per_s": world * sum(terms) / (ms / 1e3),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "frac_of_spec_8000GBs": achieved / 8000.0,
                     "kernel": ("gs::taylor2d_kernel (cooperative; one launch per step, one resident CTA per 32x32 "
                                "tile, four terms per grid barrier; L2-resident, latency-bound)" if flat2d else
                                "gs::taylor_kernel (cooperative; one launch per step, fused two-term sweeps)"),
                     "launches": taylor_n, "avg_launch_ms": taylor_ms / max(taylor_n, 1),
                     "share_of_step": taylor_ms / (pass2_ms if separate else ms),
                     "kernel_timing": ("separate pass of the same K steps inside bench.py (per-kernel events + step "
                                       f"log; {pass2_ms / args.steps:.4f} ms/step); `value` is the production path "
                                       "without them" if separate else "per-kernel events inside the timed region"),
                     "algorithmic_bytes": (("per voxel and round (4 terms): 40 B written (f after each level, T_4) + "
                                            "12.5 B box reload, all L2; "
                                            f"{taylor_bytes / max(taylor_n, 1) / 1e9:.2f} GB per launch, "
                                            f"{np.mean([x[1] for x in tb]):.1f} rounds per step") if flat2d else
                                           ("per voxel: 33 B per fused two-term sweep (25 B stage-0 first sweep) "
                                            "+ 8 B per stage started from an implicit f = F + T; "
                                            f"{taylor_bytes / max(taylor_n, 1) / 1e9:.2f} GB per launch, "
                                            f"{np.mean([x[1] for x in tb]):.1f} sweeps per step, "
                                            f"{np.mean([x[2] for x in tb]):.1f} of them implicit stage starts")),
                     "exact_reruns_per_step": float(np.mean([infos[q].reruns for q in range(args.steps)])),
                     "single_term_equivalent_GBs": single_term_equiv,
                     "single_term_note": ("SURVEY 8(d)'s 33 B/voxel per Taylor term over the same time; exceeds the "
                                          "HBM peak because each sweep applies two terms per pass (temporal blocking)")},
        "step_bytes_per_s_GBs": step_bytes / (ms / 1e3) / 1e9,
        "kernel_ms": {k: v[0] / args.steps for k, v in ktimes.items()},
        "gpu_launches": timed_launches(op, args.steps, separate),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line))
    op.close()
    if dist:
        dist.destroy_process_group()


def run_ensemble(args, w, rank, world, local):
    """C5: every bench step advances all 64 members by one exponential-Euler step; members are
    partitioned over ranks (replicas, no data-path collective); value = member-steps/s."""
    import torch
    from paper_2402_02273_b200 import ensemble as E
    from paper_2402_02273_b200 import gliosim as G
    from paper_2402_02273_b200 import workloads as W

    torch.cuda.set_device(local)
    dist = None
    if world > 1 or under_launcher():
        import torch.distributed as D
        D.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = D
    members = E.members_for_rank(w.members, rank, world)
    runner = E.EnsembleRunner(w, members, device=local)
    runner.reset()
    runner.run(args.warmup, batched=not os.environ.get("GS_ENS_SEQUENTIAL"))
    runner.reset()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    batched_run = not os.environ.get("GS_ENS_SEQUENTIAL") and bool(runner.ops)
    if batched_run:
        runner.ops[0].set_kernel_timing(True)  # CUDA events around each step's batched Taylor launch
    with Clocks(local) as clk:
        t0.record()
        results = runner.run(args.steps, batched=not os.environ.get("GS_ENS_SEQUENTIAL"))  # synchronous
        t1.record()
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    roofline = None
    if batched_run:
        taylor_ms, taylor_n = runner.ops[0].kernel_times()["taylor"]
        runner.ops[0].set_kernel_timing(False)
        if taylor_n and all(r.stage_terms is not None for r in results):
            peak, peak_kind = measured_peak()
            per_voxel = sum(taylor_bytes_per_voxel(st)[0] for r in results for st in r.stage_terms)
            sweeps = sum(taylor_bytes_per_voxel(st)[1] for r in results for st in r.stage_terms)
            tbytes = w.n * per_voxel
            achieved = tbytes / (taylor_ms / 1e3) / 1e9
            traffic = None
            try:
                with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                    tr = json.load(f).get(w.name)
                    if tr:
                        traffic = tr["taylor_dram_bytes_per_launch"]
            except Exception:
                pass
            roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "traffic": traffic, "peak_kind": peak_kind, "frac_of_spec_8000GBs": achieved / 8000.0,
                        "kernel": ("gs::ens_taylor_kernel (cooperative; one launch per ensemble step serves every "
                                   "member of this rank, 16 at a time on groups of SMs)"),
                        "launches": taylor_n, "avg_launch_ms": taylor_ms / taylor_n, "share_of_step": taylor_ms / ms,
                        "algorithmic_bytes": ("per voxel and member: 33 B per fused two-term sweep (25 B stage-0 first "
                                              "sweep) + 8 B per implicit stage start; "
                                              f"{tbytes / taylor_n / 1e9:.2f} GB per launch, "
                                              f"{sweeps / max(len(results) * args.steps, 1):.1f} sweeps per member-step")}
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    table, terms = E.gather_results(results, w.members, args.steps, dist)
    value = w.members * args.steps / (ms / 1e3)

    # e2e: the drop-in step() with host buffers for every member of this rank, one ensemble step
    e2e = None
    if not args.no_e2e:
        import ctypes as C
        from paper_2402_02273_b200 import _native as N
        # every member's input already in pinned host memory, as the contract's e2e asks
        pin_ins = []
        for u in runner.u0:
            t = torch.empty(w.n, dtype=torch.float64, pin_memory=True)
            t.numpy()[:] = u
            pin_ins.append(t)
        pin_outs = [torch.empty(w.n, dtype=torch.float64, pin_memory=True) for _ in runner.ops]
        batched = not os.environ.get("GS_ENS_SEQUENTIAL")
        info = N.GsStepInfo()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        # device-timed (events on the idle default stream bracket the synchronous calls)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if batched:
            # every member's u H2D, one batched step, every u' D2H: gs_step_ensemble_host, whose
            # member chunks' copies overlap the other chunks' steps
            G.step_ensemble_host(runner.ops, [t.numpy() for t in pin_ins], runner.rhos, w.tau, W.TOL,
                                 outs=[t.numpy() for t in pin_outs])
        else:
            for op, pin_in, pin_out, rho in zip(runner.ops, pin_ins, pin_outs, runner.rhos):
                rc = op.lib.gs_step_host(op.ctx, pin_in.numpy(), rho, w.tau, W.TOL, pin_out.numpy(), C.byref(info))
                assert rc == 0
        e1.record()
        torch.cuda.synchronize()
        dt = e0.elapsed_time(e1) / 1e3
        if dist:
            t = torch.tensor([dt], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": w.members / dt, "unit": "member-steps/s", "h2d_bytes_per_step": 8 * w.n * w.members,
               "d2h_bytes_per_step": 8 * w.n * w.members,
               "api": ("gs_step_ensemble_host: every member's u H2D from pinned, one batched step, u' D2H; 4 member "
                       "chunks whose copies overlap the other chunks' steps" if batched else
                       "gs_step_host per member (drop-in step(): u H2D from pinned, u' D2H)")}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sample = cpu_reference_sample(w, runner.ops[0].labels(), runner.u0[0], 50, rho=runner.rhos[0],
                                          budget_s=args.cpu_seconds)
            cpu = {"value": 1.0 / float(np.mean(sample["step_times"])), "unit": "member-steps/s",
                   "cores": sample["cores"], "kind": sample["kind"],
                   "sample": (f"{sample['steps']} gliosim::run steps (workers={sample['cores']}) of member 0 "
                              f"(128^3, rho={runner.rhos[0]:.4f}); one member-step each")}
        except Exception as e:
            cpu = {"value": None, "unit": "member-steps/s", "cores": os.cpu_count(), "kind": "unavailable",
                   "sample": f"failed: {e}"}
    line = {
        "metric": "ensemble member-steps/s (64 x 128^3 fp64)", "value": value, "unit": "member-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded shell phantoms, one per member)",
        "config": {"workload": f"{w.name}: {w.note}", "members": w.members, "grid": [w.nx, w.ny, w.nz],
                   "members_per_rank": len(members), "parallelism": f"members partitioned over {world} rank(s)",
                   "batching": ("gs_run_ensemble: one launch per kernel of the step for all members; the Taylor "
                                "launch runs 16 members at a time on groups of 9 SMs, longest members first"
                                if not os.environ.get("GS_ENS_SEQUENTIAL") else "sequential gs_run per member"),
                   "terms_per_member_step": float(terms.mean()),
                   "rho_range": [float(min(runner.rhos)), float(max(runner.rhos))] if world == 1 else None,
                   "l2": "64 resident members x 7 x 16 MiB >> L2"},
        # per batched step: prep, border, order, Taylor, update and the two passes of each exact sum
        "gpu_launches": ((5 if os.environ.get("GS_TREE_SUMS") else 9) * args.steps + 1)
        if not os.environ.get("GS_ENS_SEQUENTIAL")
        else 4 * len(members) * args.steps + len(members),
        "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu, "clocks": clk.summary(),
        "metrics_all_finite": bool(np.isfinite(table).all()),
    }
    if rank == 0:
        print(json.dumps(line))
    runner.close()
    if dist:
        dist.destroy_process_group()


def run_reference(args, w, rank, world, local):
    """The UNMODIFIED reference (oracle/_ref: gliosim compiled from /root/reference/proj/src)
    on the host cores; rank 0 only (other ranks exit)."""
    if rank != 0:
        return
    from paper_2402_02273_b200 import workloads as W
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Port
    port = Port()
    member = 0
    data, dims, labels = build_case(w)
    if labels is None:
        labels = port.resample(data, dims[0], dims[1], dims[2], (w.nx, w.ny, w.nz))
    d = np.array([0.0, W.D_WHITE, W.D_GRAY, 0.0])[labels]
    # u0 with the reference's own seed_initial (libm), max over seeds
    u0 = None
    for c in W.seed_points(w, labels, member):
        ui = port.seed_initial((w.nx, w.ny, w.nz), w.h, 1.0, W.seed_width(w), c, d)
        u0 = ui if u0 is None else np.maximum(u0, ui)
    rho = W.member_rho(w, member)
    # the reference has no warm-up effects (no JIT, no caches across run() calls): one untimed
    # step at most; the timed steps are capped by --ref-budget seconds (the first step's time
    # decides how many fit), and the line reports the number actually timed
    warm = min(args.warmup, 1)
    sample = cpu_reference_sample(w, labels, u0, args.steps, warmup=warm, rho=rho, budget_s=args.ref_budget)
    t = float(np.mean(sample["step_times"]))
    if w.members > 1:
        v = 1.0 / t
        metric, unit = "ensemble member-steps/s (64 x 128^3 fp64)", "member-steps/s"
        ms_step = 1e3 * w.members * t
        desc = (f"{sample['steps']} timed gliosim::run steps (+{warm} untimed) of member 0 on its full "
                f"{w.nx}x{w.ny}x{w.nz} grid (rho={rho:.4f}, workers={sample['cores']}); member-steps/s")
    else:
        v = 1.0 / t
        metric = "expEuler steps/s at 256^3 fp64" if w.name.startswith("C4") else f"expEuler steps/s ({w.name})"
        unit = "steps/s"
        ms_step = 1e3 * t
        desc = (f"{sample['steps']} timed gliosim::run steps (+{warm} untimed) of the full {w.nx}x{w.ny}x{w.nz} grid "
                f"(workers={sample['cores']}), {t:.2f} s/step, RunTimings::step_seconds")
    line = {
        "impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": world, "steps": sample["steps"],
        "steps_requested": args.steps, "step_seconds": sample["step_times"],
        "warmup": warm, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if w.members > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded shell phantom, BASELINE.json config)",
        "config": {"workload": f"{w.name}: {w.note}", "grid": [w.nx, w.ny, w.nz], "parallelism": "CPU threads"},
        "cpu_baseline": {"value": v, "unit": unit, "cores": sample["cores"], "kind": sample["kind"], "sample": desc},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    args = parse()
    rank, world, local = dist_env()
    from paper_2402_02273_b200 import workloads as W
    w = W.get(args.config)
    if args.steps is None:
        args.steps = 10 if (args.impl == "reference" or w.n >= 256 ** 3) else w.steps
    if args.impl == "reference":
        run_reference(args, w, rank, world, local)
    elif w.members > 1:
        run_ensemble(args, w, rank, world, local)
    else:
        run_ours(args, w, rank, world, local)


if __name__ == "__main__":
    main()

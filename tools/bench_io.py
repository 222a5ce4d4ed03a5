"""Measure the SURVEY.md 8(f) #2 / #4 rows on a B200 box (prints JSON lines).

  python tools/bench_io.py [--out profiles/r01_io_bench.json]

1. snapshot I/O: C4 (256^3) run_to_directory, 4 steps with a snapshot every 2 steps
   (nodes 0, 2, 4), against the same 4 steps with no sink.  Reports the wall-clock cost
   per snapshot that the asynchronous sink leaves exposed, and the native writer's
   throughput on one 256^3 state (gs_write_vtk, all host threads), next to the reference's
   own write_vtk on the same state (oracle/_ref, when present).
2. ingest: a 532x565x29 PGM stack (the paper's scan size) -> load_stack -> resample +
   classify on the GPU to 256^3, against the reference's load_stack + resample (CPU).
"""
import argparse
import json
import os
import shutil
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2402_02273_b200 import gliosim as G, phantom, workloads as W  # noqa: E402


def ref_lib():
    try:
        from oracle import Ref, REF_SO
        return Ref(REF_SO) if os.path.exists(REF_SO) else None
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--skip-ref", action="store_true")
    args = ap.parse_args()
    lines = []
    tmp = tempfile.mkdtemp(prefix="gs_io_")
    ref = None if args.skip_ref else ref_lib()
    try:
        w = W.get("C4")
        data, wd, ht, sl = W.intensity(w)
        grid = G.Grid(w.nx, w.ny, w.nz, w.h)
        op = G.StencilOperator.from_intensity(grid, data, wd, ht, sl)
        labels = op.labels()
        c = W.seed_points(w, labels)[0]
        cfg = G.SimConfig(nx=w.nx, ny=w.ny, nz=w.nz, h=w.h, t0=W.T0, t_end=W.T0 + 4 * W.TAU, num_steps=4,
                          snapshot_every=2, seed_center=c, seed_amplitude=1.0, seed_width=W.seed_width(w))
        u0 = G.seed_initial(op, cfg)
        G.run(cfg, op, u0)  # warm
        t = time.perf_counter()
        r0 = G.run(cfg, op, u0)
        plain = time.perf_counter() - t
        out_dir = os.path.join(tmp, "run")
        G.run_to_directory(cfg, op, labels, out_dir)  # warm (allocates the slots)
        t = time.perf_counter()
        r1 = G.run_to_directory(cfg, op, labels, out_dir)
        with_io = time.perf_counter() - t
        assert np.array_equal(r0.u, r1.u)
        size = os.path.getsize(os.path.join(out_dir, "snapshot_0004.vtk"))
        # one snapshot through the synchronous native writer, all host threads
        state = r1.u
        t = time.perf_counter()
        G.write_vtk(G.ScalarField(grid, state), os.path.join(tmp, "one.vtk"), labels)
        native = time.perf_counter() - t
        t = time.perf_counter()
        G.write_vtk(G.ScalarField(grid, state), "/dev/null", labels)  # formatting alone, no file system
        fmt_only = time.perf_counter() - t
        # one snapshot of the resident state through the asynchronous sink (GPU formatter), to flush
        op.set_state(state)
        op.snapshot_vtk(os.path.join(tmp, "warm.vtk"), labels)
        op.flush_snapshots()
        t = time.perf_counter()
        op.snapshot_vtk(os.path.join(tmp, "gpu.vtk"), labels)
        t_call = time.perf_counter() - t
        op.flush_snapshots()
        gpu_snap = time.perf_counter() - t
        t = time.perf_counter()
        G.seed_initial(op, cfg)
        seed_s = time.perf_counter() - t
        line = {"bench": "snapshot_io", "workload": "C4 256^3, 4 steps, snapshot_every 2 (3 snapshots + csv)",
                "gpu_formatted_snapshot_s": round(gpu_snap, 4), "snapshot_call_returns_after_s": round(t_call, 5),
                "seed_initial_s": round(seed_s, 4),
                "run_s": round(plain, 4), "run_to_directory_s": round(with_io, 4),
                "exposed_s_per_snapshot": round((with_io - plain) / 3, 4),
                "snapshot_bytes": size, "native_write_vtk_s": round(native, 4),
                "native_values_per_s": round(w.n / native, 1), "format_only_s": round(fmt_only, 4),
                "host_threads": os.cpu_count()}
        if ref is not None:
            t = time.perf_counter()
            ref.write_vtk(os.path.join(tmp, "ref.vtk"), state, (w.nx, w.ny, w.nz), w.h, (0.0, 0.0, 0.0), labels)
            rs = time.perf_counter() - t
            with open(os.path.join(tmp, "ref.vtk"), "rb") as a, open(os.path.join(tmp, "one.vtk"), "rb") as b, \
                    open(os.path.join(tmp, "gpu.vtk"), "rb") as g:
                ra = a.read()
                same = ra == b.read()
                line["gpu_bytes_identical"] = ra == g.read()
            line.update({"reference_write_vtk_s": round(rs, 4), "bytes_identical": same,
                         "speedup_vs_reference_writer": round(rs / native, 1)})
        t = time.perf_counter()
        back = G.read_vtk(os.path.join(tmp, "one.vtk"))
        line["native_read_vtk_s"] = round(time.perf_counter() - t, 4)
        line["read_back_bitwise"] = bool(np.array_equal(back.values.view(np.uint64), state.view(np.uint64)))
        lines.append(line)
        op.close()

        # ---- ingest: 532 x 565 x 29 PGM stack -> 256^3 labels on the GPU ----------------
        ws, hs, ns = 532, 565, 29
        stack = phantom.slice_stack(ws, hs, ns, 160, seed=7)
        paths = []
        for s in range(ns):
            p = os.path.join(tmp, f"slice_{s:03d}.pgm")
            with open(p, "wb") as f:
                f.write(f"P5\n{ws} {hs}\n255\n".encode() + stack[s].tobytes())
            paths.append(p)
        g256 = G.Grid(256, 256, 256, 200.0 / 255.0)
        best = None
        for _ in range(3):
            t = time.perf_counter()
            st = G.load_stack(paths)
            t_load = time.perf_counter() - t
            t = time.perf_counter()
            with G.stencil_from_stack(st, g256) as op2:
                lab = op2.labels()
            t_map = time.perf_counter() - t
            best = min(best or (9e9, 0, 0), (t_load + t_map, t_load, t_map))
        line = {"bench": "ingest", "workload": "532x565x29 PGM stack -> 256^3 material map + D palette",
                "total_s": round(best[0], 4), "load_stack_s": round(best[1], 4),
                "resample_classify_upload_s": round(best[2], 4)}
        if ref is not None:
            t = time.perf_counter()
            dims, inten = ref.load_stack(paths)
            t_rl = time.perf_counter() - t
            t = time.perf_counter()
            rl = ref.resample(inten, *dims, (256, 256, 256))
            t_rr = time.perf_counter() - t
            line.update({"reference_load_stack_s": round(t_rl, 4), "reference_resample_s": round(t_rr, 4),
                         "labels_identical": bool(np.array_equal(rl, lab))})
        lines.append(line)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    for ln in lines:
        print(json.dumps(ln))
    if args.out:
        with open(args.out, "w") as f:
            for ln in lines:
                f.write(json.dumps(ln) + "\n")


if __name__ == "__main__":
    main()

"""Summarise one `ncu --set full` capture of taylor_kernel into a text file for profiles/.

  python tools/ncu_summary.py gpurun_out/m_taylor.ncu-rep profiles/r01_taylor_ncu_summary.txt \
      --title "round 1" --peak 6537 --alg-gb 50.59 [--traffic-json profiles/ncu_traffic.json --config C4]

Reads the report here (ncu -i ... --csv); no GPU needed.
"""
import argparse
import csv
import io
import json
import subprocess

CMD = ("ncu --set full --clock-control none --import-source on -k regex:taylor_kernel -s 1 -c 1 "
       "python tools/prof_step.py --config C4 --steps 1 --repeat 2")
STALLS = ["wait", "barrier", "not_selected", "selected", "long_scoreboard", "math_pipe_throttle",
          "short_scoreboard", "branch_resolving", "dispatch_stall", "no_instructions", "mio_throttle",
          "lg_throttle", "membar", "sleeping", "tex_throttle", "drain", "misc", "imc_miss"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True, check=True)
    return list(csv.reader(io.StringIO(out.stdout)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--title", default="")
    ap.add_argument("--peak", type=float, required=True, help="measured HBM copy peak, GB/s")
    ap.add_argument("--alg-gb", type=float, default=None, help="algorithmic GB per launch (bench.py)")
    ap.add_argument("--traffic-json", default=None)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--kernel-desc", default="taylor_kernel<2> (C4 256^3, one exponential-Euler step = 1 launch)")
    ap.add_argument("--command", default=CMD)
    a = ap.parse_args()

    lines = [f"# ncu --set full, {a.kernel_desc}, {a.title}", f"# command: {a.command}", ""]
    det = ncu_csv(a.rep, "details")
    h = det[0]
    si, mi, ui, vi = (h.index(k) for k in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    for row in det[1:]:
        lines.append(f"{row[si]} | {row[mi]} | {row[vi]} {row[ui]}".rstrip())
    raw = ncu_csv(a.rep, "raw")
    d = dict(zip(raw[0], raw[2]))
    units = dict(zip(raw[0], raw[1]))  # the raw page scales each metric: Kbyte / Mbyte / Gbyte, us / ms
    scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
             "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    f = lambda k: float(d[k]) * scale.get(units.get(k, ""), 1.0)  # noqa: E731  (GB and ms)
    dur_ms = f("gpu__time_duration.sum")
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "lts__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"):
        if k in d:
            lines.append(f"raw | {k} | {d[k]} {raw[1][raw[0].index(k)]}".rstrip())
    st = {}
    for s in STALLS:
        k = f"smsp__pcsamp_warps_issue_stalled_{s}"
        if k in d and d[k] not in ("", "n/a"):
            st[s] = float(d[k])
    tot = sum(st.values()) or 1.0
    for s, x in sorted(st.items(), key=lambda t: -t[1]):
        if x / tot >= 0.01:
            lines.append(f"stall share | {s} | {x / tot:.3f}")
    gb = rd + wr
    lines.append(f"derived | DRAM bytes per launch | {gb:.2f} GB; {gb / dur_ms:.3f} TB/s = "
                 f"{gb / dur_ms * 1e3 / a.peak:.3f} of the measured {a.peak:.0f} GB/s copy peak")
    if a.alg_gb:
        lines.append(f"derived | algorithmic bytes per launch (bench.py) | {a.alg_gb:.2f} GB; DRAM/algorithmic "
                     f"{gb / a.alg_gb:.3f}; algorithmic {a.alg_gb / dur_ms:.3f} TB/s = "
                     f"{a.alg_gb / dur_ms * 1e3 / a.peak:.3f} of peak (cold-cache, serialised ncu timing)")
    with open(a.out, "w") as fo:
        fo.write("\n".join(lines) + "\n")
    if a.traffic_json:
        try:
            with open(a.traffic_json) as fi:
                tj = json.load(fi)
        except FileNotFoundError:
            tj = {}
        tj[a.config] = {"taylor_dram_bytes_per_launch": gb * 1e9, "read": rd * 1e9, "write": wr * 1e9,
                        "source": f"{a.out} (ncu --set full, one taylor_kernel launch = one step)"}
        with open(a.traffic_json, "w") as fo:
            json.dump(tj, fo, indent=1)
            fo.write("\n")


if __name__ == "__main__":
    main()

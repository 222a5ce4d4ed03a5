# Per-kernel durations of one step (ncu launch list, second launch) for each config given:
#   bash tools/launch_list.sh C4 C2   (on the GPU box; prints "config kernel ns")
mkdir -p gpurun_out
for c in "$@"; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$c.csv \
      python tools/prof_step.py --config $c --steps 1 --repeat 2 > /dev/null 2>&1
  python - "$c" <<'PY'
import csv, sys
c = sys.argv[1]
rows = [r for r in csv.DictReader(l for l in open(f"gpurun_out/ll_{c}.csv") if not l.startswith("=="))]
for r in rows[len(rows) // 2:]:
    print(c, r["Kernel Name"][:44], r["Metric Value"])
PY
done

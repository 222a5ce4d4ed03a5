# Copy a round_measure.sh batch from gpurun_out/ into profiles/ (run here, no GPU):
#   bash tools/round_collect.sh r01
set -eu
r=${1:-r01}
tail -1 gpurun_out/m_bench.json > profiles/${r}_bench_c4.json
tail -1 gpurun_out/m_bench_ref.json > profiles/${r}_bench_reference_c4.json
cp gpurun_out/m_launches.csv profiles/${r}_launches_c4.csv
for c in C1 C2 C3 C5 C4x4; do tail -1 gpurun_out/cfg_$c.json > profiles/${r}_bench_$c.json; done
# the ncu summaries and the DRAM traffic were written on the GPU box (round_measure.sh)
cp gpurun_out/m_taylor_ncu_summary.txt profiles/${r}_taylor_ncu_summary.txt
for k in taylor_c3 ens_taylor taylor2d_c2; do
  [ -f gpurun_out/m_${k}_ncu_summary.txt ] && cp gpurun_out/m_${k}_ncu_summary.txt profiles/${r}_${k}_ncu_summary.txt
done
python - "$r" <<'PY'
import json, sys
r = sys.argv[1]
t = json.load(open("gpurun_out/m_ncu_traffic.json"))
names = {"C4": "taylor", "C3": "taylor_c3", "C5": "ens_taylor", "C2": "taylor2d_c2"}
for c, v in t.items():
    if c in names:
        v["source"] = f"profiles/{r}_{names[c]}_ncu_summary.txt (ncu --set full, one Taylor launch = one step)"
json.dump(t, open("profiles/ncu_traffic.json", "w"), indent=1)
open("profiles/ncu_traffic.json", "a").write("\n")
PY
cuobjdump -sass -fun '_ZN2gs13taylor_kernelILi2EEEvNS_11SolveParamsEii' paper_2402_02273_b200/libgliosim_b200.so 2>/dev/null \
    | gzip -9 > profiles/${r}_taylor_kernel.sass.gz
echo "collected into profiles/ (${r}_*)"

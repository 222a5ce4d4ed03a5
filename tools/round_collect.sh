# Copy a round_measure.sh batch from gpurun_out/ into profiles/ (run here, no GPU):
#   bash tools/round_collect.sh r01
set -eu
r=${1:-r01}
tail -1 gpurun_out/m_bench.json > profiles/${r}_bench_c4.json
tail -1 gpurun_out/m_bench_ref.json > profiles/${r}_bench_reference_c4.json
cp gpurun_out/m_launches.csv profiles/${r}_launches_c4.csv
for c in C1 C2 C3 C5 C4x4; do tail -1 gpurun_out/cfg_$c.json > profiles/${r}_bench_$c.json; done
alg=$(python -c "import json,re; d=json.load(open('profiles/${r}_bench_c4.json')); print(re.search(r'([0-9.]+) GB per launch', d['roofline']['algorithmic_bytes']).group(1))")
python tools/ncu_summary.py gpurun_out/m_taylor.ncu-rep profiles/${r}_taylor_ncu_summary.txt --title "$r" --peak \
    "$(python -c "import json; print(json.load(open('MEASURED_PEAKS.json'))['hbm_gbs'])")" --alg-gb "$alg" \
    --traffic-json profiles/ncu_traffic.json --config C4
peak=$(python -c "import json; print(json.load(open('MEASURED_PEAKS.json'))['hbm_gbs'])")
algof() { python -c "import json,re; d=json.load(open('profiles/${r}_bench_$1.json')); print(re.search(r'([0-9.]+) GB per launch', d['roofline']['algorithmic_bytes']).group(1))"; }
[ -f gpurun_out/m_taylor_c3.ncu-rep ] && python tools/ncu_summary.py gpurun_out/m_taylor_c3.ncu-rep profiles/${r}_taylor_c3_ncu_summary.txt \
    --title "$r" --peak "$peak" --alg-gb "$(algof C3)" --traffic-json profiles/ncu_traffic.json --config C3 \
    --kernel-desc "taylor_kernel<2> (C3 128^3, one exponential-Euler step = 1 launch)" \
    --command "ncu --set full --clock-control none --import-source on -k regex:taylor_kernel -s 1 -c 1 python tools/prof_step.py --config C3 --steps 1 --repeat 2"
[ -f gpurun_out/m_taylor_c5.ncu-rep ] && python tools/ncu_summary.py gpurun_out/m_taylor_c5.ncu-rep profiles/${r}_ens_taylor_ncu_summary.txt \
    --title "$r" --peak "$peak" --alg-gb "$(algof C5)" --traffic-json profiles/ncu_traffic.json --config C5 \
    --kernel-desc "ens_taylor_kernel<2> (C5: 64 x 128^3, one batched ensemble step = 1 launch)" \
    --command "ncu --set full --clock-control none --import-source on -k regex:ens_taylor -s 1 -c 1 python tools/prof_ens.py"
[ -f gpurun_out/m_taylor_c2.ncu-rep ] && python tools/ncu_summary.py gpurun_out/m_taylor_c2.ncu-rep profiles/${r}_taylor2d_c2_ncu_summary.txt \
    --title "$r" --peak "$peak" --alg-gb "$(algof C2)" \
    --kernel-desc "taylor2d_kernel (C2 256^2, one exponential-Euler step = 1 launch)" \
    --command "ncu --set full --clock-control none --import-source on -k regex:taylor2d -s 1 -c 1 python tools/prof_step.py --config C2 --steps 1 --repeat 2"
cuobjdump -sass -fun '_ZN2gs13taylor_kernelILi2EEEvNS_11SolveParamsEii' paper_2402_02273_b200/libgliosim_b200.so 2>/dev/null \
    | gzip -9 > profiles/${r}_taylor_kernel.sass.gz
echo "collected into profiles/ (${r}_*)"

# Round-end measurement batch (run on the GPU box from the repo root):
#   bash tools/round_measure.sh          (then, here: bash tools/round_collect.sh rNN)
# GPU tests, smoke(), the C4 bench line (both arms), the ncu launch list of the same default bench
# command, one ncu --set full capture of the Taylor kernel (each ncu pass only after its command
# exited 0), and the bench lines of the other configurations.
set -u
mkdir -p gpurun_out
[ -n "${SKIP_TESTS:-}" ] || { timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/m_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/m_tests.log; }
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/m_smoke.log
timeout 900 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/m_bench_ref.json 2> gpurun_out/m_bench_ref.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m_launches.csv \
    python bench.py > gpurun_out/m_ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 python tools/prof_step.py --config C4 --steps 1 --repeat 2 > gpurun_out/m_prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:taylor_kernel -s 1 -c 1 \
    -o gpurun_out/m_taylor python tools/prof_step.py --config C4 --steps 1 --repeat 2 > gpurun_out/m_ncu_full.log 2>&1; echo "full rc=$?"
# the same capture for the 128^3 Taylor path (C3), the batched ensemble (C5) and the 2-D kernel (C2)
timeout 600 python tools/prof_step.py --config C3 --steps 1 --repeat 2 > gpurun_out/m_prof_c3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:taylor_kernel -s 1 -c 1 \
    -o gpurun_out/m_taylor_c3 python tools/prof_step.py --config C3 --steps 1 --repeat 2 > gpurun_out/m_ncu_c3.log 2>&1; echo "full C3 rc=$?"
timeout 600 python tools/prof_ens.py > gpurun_out/m_prof_c5.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ens_taylor -s 1 -c 1 \
    -o gpurun_out/m_taylor_c5 python tools/prof_ens.py > gpurun_out/m_ncu_c5.log 2>&1; echo "full C5 rc=$?"
timeout 600 python tools/prof_step.py --config C2 --steps 1 --repeat 2 > gpurun_out/m_prof_c2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:taylor2d -s 1 -c 1 \
    -o gpurun_out/m_taylor_c2 python tools/prof_step.py --config C2 --steps 1 --repeat 2 > gpurun_out/m_ncu_c2.log 2>&1; echo "full C2 rc=$?"
bash tools/configs_measure.sh C1 C2 C3 C5 C4x4
# summarise the captures here (ncu reads them without a GPU too, but four reports with source
# exceed what gpurun brings back): text summaries + DRAM traffic into gpurun_out/, then only
# the C4 report travels
peak=$(python -c "import json; print(json.load(open('MEASURED_PEAKS.json'))['hbm_gbs'])" 2>/dev/null || echo 6429)
algof() { python -c "import json,re; d=json.loads(open('gpurun_out/$1').read().strip().splitlines()[-1]); print(re.search(r'([0-9.]+) GB per launch', d['roofline']['algorithmic_bytes']).group(1))"; }
cp profiles/ncu_traffic.json gpurun_out/m_ncu_traffic.json 2>/dev/null
sum1() {  # rep out config alg-json kernel-desc command
  [ -f "$1" ] && python tools/ncu_summary.py "$1" "gpurun_out/$2" --title "${ROUND:-r02}" --peak "$peak" --alg-gb "$(algof $4)" \
      --traffic-json gpurun_out/m_ncu_traffic.json --config "$3" --kernel-desc "$5" --command "$6"
}
sum1 gpurun_out/m_taylor.ncu-rep m_taylor_ncu_summary.txt C4 m_bench.json "taylor_kernel<2> (C4 256^3, one exponential-Euler step = 1 launch)" \
  "ncu --set full --clock-control none --import-source on -k regex:taylor_kernel -s 1 -c 1 python tools/prof_step.py --config C4 --steps 1 --repeat 2"
sum1 gpurun_out/m_taylor_c3.ncu-rep m_taylor_c3_ncu_summary.txt C3 cfg_C3.json "taylor_kernel<2> (C3 128^3, one exponential-Euler step = 1 launch)" \
  "ncu --set full --clock-control none --import-source on -k regex:taylor_kernel -s 1 -c 1 python tools/prof_step.py --config C3 --steps 1 --repeat 2"
sum1 gpurun_out/m_taylor_c5.ncu-rep m_ens_taylor_ncu_summary.txt C5 cfg_C5.json "ens_taylor_kernel<2> (C5: 64 x 128^3, one batched ensemble step = 1 launch)" \
  "ncu --set full --clock-control none --import-source on -k regex:ens_taylor -s 1 -c 1 python tools/prof_ens.py"
sum1 gpurun_out/m_taylor_c2.ncu-rep m_taylor2d_c2_ncu_summary.txt C2 cfg_C2.json "taylor2d_kernel (C2 256^2, one exponential-Euler step = 1 launch)" \
  "ncu --set full --clock-control none --import-source on -k regex:taylor2d -s 1 -c 1 python tools/prof_step.py --config C2 --steps 1 --repeat 2"
rm -f gpurun_out/m_taylor_c3.ncu-rep gpurun_out/m_taylor_c5.ncu-rep gpurun_out/m_taylor_c2.ncu-rep
du -sh gpurun_out
[ -f gpurun_out/m_tests.log ] && tail -3 gpurun_out/m_tests.log

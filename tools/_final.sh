bash tools/round_measure.sh
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/m_smoke.log
bash tools/configs_measure.sh C1 C2 C3 C4x4

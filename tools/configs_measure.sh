# Bench lines for the non-headline configs (run on the GPU box from the repo root):
#   bash tools/configs_measure.sh [C1 C2 C3 C5 C4x4]
mkdir -p gpurun_out
cfgs=${*:-C1 C2 C3 C5 C4x4}
for c in $cfgs; do
  timeout 900 python bench.py --config $c > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; echo "$c rc=$?"
done

# A/B timing of library variants on one box: bash tools/abrun.sh name=lib[:ENV=VAL] ...
# Each variant's .so is copied over the in-tree library and bench.py runs C4 (20 steps), twice.
mkdir -p gpurun_out
cp paper_2402_02273_b200/libgliosim_b200.so /tmp/gs_lib_keep.so
for rep in 1 2; do
  for spec in "$@"; do
    name=${spec%%=*}; rest=${spec#*=}; lib=${rest%%:*}; envs=""
    [ "$rest" != "$lib" ] && envs=${rest#*:}
    cp "$lib" paper_2402_02273_b200/libgliosim_b200.so
    env $envs timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],2), round(d['roofline']['avg_launch_ms'],3), 'terms', d['config']['terms_per_step'], 'reruns', d['roofline']['exact_reruns_per_step'])"
  done
done
cp /tmp/gs_lib_keep.so paper_2402_02273_b200/libgliosim_b200.so

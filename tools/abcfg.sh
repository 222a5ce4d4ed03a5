# bash tools/abcfg.sh CONFIG name=lib[:ENV=VAL] ... : like abrun.sh for another workload
cfg=$1; shift
cp paper_2402_02273_b200/libgliosim_b200.so /tmp/gs_lib_keep.so
for rep in 1 2; do
  for spec in "$@"; do
    name=${spec%%=*}; rest=${spec#*=}; lib=${rest%%:*}; envs=""
    [ "$rest" != "$lib" ] && envs=${rest#*:}
    cp "$lib" paper_2402_02273_b200/libgliosim_b200.so
    env $envs timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $name', round(d['value'],1), d.get('kernel_ms'))"
  done
done
cp /tmp/gs_lib_keep.so paper_2402_02273_b200/libgliosim_b200.so

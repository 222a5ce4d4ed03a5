# bash tools/ncu_dram.sh name=lib[:ENV=VAL] ... : DRAM bytes, L2 hit rate and duration of one
# taylor_kernel launch (C4) per library variant, from ncu (counters only, not a timing run).
cp paper_2402_02273_b200/libgliosim_b200.so /tmp/gs_lib_keep.so
cfg=${CFG:-C4}
for spec in "$@"; do
  name=${spec%%=*}; rest=${spec#*=}; lib=${rest%%:*}; envs=""
  [ "$rest" != "$lib" ] && envs=${rest#*:}
  cp "$lib" paper_2402_02273_b200/libgliosim_b200.so
  env $envs timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
    --clock-control none -k regex:taylor_kernel -s 1 -c 1 --csv python tools/prof_step.py --config $cfg --steps 1 --repeat 2 2>/dev/null \
    | grep -E '"(dram__|lts__|gpu__)' | awk -F'","' -v n="$name" '{gsub(/"/,"",$NF); print n, $(NF-2), $NF}'
done
cp /tmp/gs_lib_keep.so paper_2402_02273_b200/libgliosim_b200.so

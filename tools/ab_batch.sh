# One GPU call: parity of variant libraries, then A/B timings (bash tools/ab_batch.sh v3 v4 ...)
# Variants are build_ab/lib_<name>.so; build_ab/lib_base.so is the reference point.
mkdir -p gpurun_out
cp paper_2402_02273_b200/libgliosim_b200.so /tmp/gs_lib_orig.so
for v in "$@"; do
  cp build_ab/lib_$v.so paper_2402_02273_b200/libgliosim_b200.so
  touch paper_2402_02273_b200/libgliosim_b200.so
  timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_ensemble.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/ab_parity_$v.log 2>&1
  echo "parity $v rc=$? $(tail -1 gpurun_out/ab_parity_$v.log)"
done
cp /tmp/gs_lib_orig.so paper_2402_02273_b200/libgliosim_b200.so
specs="base=build_ab/lib_base.so"
for v in "$@"; do specs="$specs $v=build_ab/lib_$v.so"; done
bash tools/abrun.sh $specs
bash tools/abcfg.sh C3 $specs
bash tools/abcfg.sh C5 $specs

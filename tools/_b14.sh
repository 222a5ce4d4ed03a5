timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_ensemble.py tests/test_gpu_fullsize.py -m gpu -q -x -k "not cpp_dropin" > gpurun_out/b14_tests.log 2>&1; echo "rc=$?" >> gpurun_out/b14_tests.log
bash tools/abrun.sh base=paper_2402_02273_b200/lib_base.so ring160=paper_2402_02273_b200/lib_new.so > gpurun_out/b14_ab.log 2>&1

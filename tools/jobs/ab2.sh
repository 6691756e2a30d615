mkdir -p gpurun_out
export AB_WORKLOADS=stack64k,tiny4m
python tools/ab_time.py build_ab/libveil_prev.so paper_2405_13364_b200/libveil.so > gpurun_out/ab2.log 2>&1; cat gpurun_out/ab2.log
python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_checked_build_gpu.py > gpurun_out/ab2_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/ab2_tests.log

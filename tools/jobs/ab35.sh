mkdir -p gpurun_out/ab35
AB_WORKLOADS=stack64k,boxes1080,tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AC.so build_ab/libveil_AD.so > gpurun_out/ab35/ab.log 2>&1; cat gpurun_out/ab35/ab.log
python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_depth_filter.py tests/test_gpu_report.py > gpurun_out/ab35/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab35/tests.log

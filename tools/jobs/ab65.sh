mkdir -p gpurun_out/ab65
AB_WORKLOADS=stack64k,boxes1080,tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AV.so build_ab/libveil_BB.so > gpurun_out/ab65/ab.log 2>&1; cat gpurun_out/ab65/ab.log
python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_report.py tests/test_gpu_depth_filter.py > gpurun_out/ab65/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab65/tests.log

mkdir -p gpurun_out
AB_WORKLOADS=tiny4m,mixed16m,stack64k python tools/ab_time.py build_ab/libveil_G.so build_ab/libveil_H.so > gpurun_out/ab10.log 2>&1; cat gpurun_out/ab10.log
python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py > gpurun_out/ab10_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab10_tests.log

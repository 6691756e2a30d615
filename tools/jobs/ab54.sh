mkdir -p gpurun_out/ab54
AB_WORKLOADS=stack64k,boxes1080,tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AR.so build_ab/libveil_AT.so > gpurun_out/ab54/ab.log 2>&1; cat gpurun_out/ab54/ab.log
python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py > gpurun_out/ab54/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab54/tests.log

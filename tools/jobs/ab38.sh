mkdir -p gpurun_out/ab38
AB_WORKLOADS=stack64k,boxes1080,tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AD.so build_ab/libveil_AF.so > gpurun_out/ab38/ab.log 2>&1; cat gpurun_out/ab38/ab.log
python -m pytest -q -x -p no:cacheprovider tests -m gpu > gpurun_out/ab38/tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/ab38/tests.log

mkdir -p gpurun_out/ab63
AB_WORKLOADS=stack64k,boxes1080,tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AV.so build_ab/libveil_AZ.so > gpurun_out/ab63/ab.log 2>&1; cat gpurun_out/ab63/ab.log
python -m pytest -q -x -p no:cacheprovider tests -m gpu > gpurun_out/ab63/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab63/tests.log

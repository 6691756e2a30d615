mkdir -p gpurun_out
AB_WORKLOADS=tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_prevI.so build_ab/libveil_I.so > gpurun_out/ab11.log 2>&1; cat gpurun_out/ab11.log
python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "tiny or soup or dense or segment or 300" > gpurun_out/ab11_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab11_tests.log

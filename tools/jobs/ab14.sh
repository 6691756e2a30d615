mkdir -p gpurun_out
AB_WORKLOADS=stack64k,tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_prevL.so build_ab/libveil_L.so > gpurun_out/ab14.log 2>&1; cat gpurun_out/ab14.log
python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_depth_filter.py tests/test_gpu_report.py tests/test_gpu_abuffer_fullsize.py > gpurun_out/ab14_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/ab14_tests.log
VEIL_FUSED=1 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py > gpurun_out/ab14_fused.log 2>&1; echo fused rc=$?; tail -2 gpurun_out/ab14_fused.log

mkdir -p gpurun_out
for i in 1 2; do AB_WORKLOADS=stack64k python tools/ab_time.py build_ab/libveil_prevK.so build_ab/libveil_K.so; done > gpurun_out/ab13.log 2>&1; cat gpurun_out/ab13.log
python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_depth_filter.py tests/test_gpu_report.py > gpurun_out/ab13_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/ab13_tests.log

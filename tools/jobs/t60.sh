python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_depth_filter.py > gpurun_out/t60.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/t60.log

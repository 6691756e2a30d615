mkdir -p gpurun_out
python -m pytest -q -p no:cacheprovider tests/test_multi_device_gpu.py tests/test_gpu_fullsize.py tests/test_multirank_gpu.py tests/test_gpu_report.py tests/test_cli.py > gpurun_out/multi1.log 2>&1; echo rc=$?; tail -15 gpurun_out/multi1.log
VEIL_FUSED=1 python -m pytest -q -p no:cacheprovider tests/test_gpu_fullsize.py tests/test_multi_device_gpu.py > gpurun_out/multi1_fused.log 2>&1; echo fused rc=$?; tail -5 gpurun_out/multi1_fused.log

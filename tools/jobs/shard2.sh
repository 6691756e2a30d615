mkdir -p gpurun_out
python -m pytest -q -p no:cacheprovider tests/test_multi_device_gpu.py tests/test_multirank_gpu.py tests/test_checked_build_gpu.py tests/test_gpu_parity.py -k "shard or multi or checked or rank" > gpurun_out/shard2.log 2>&1; echo rc=$?; tail -3 gpurun_out/shard2.log
python tools/shard_sweep.py stack64k tiny4m mixed16m > gpurun_out/shard_sweep2.log 2>&1; cat gpurun_out/shard_sweep2.log

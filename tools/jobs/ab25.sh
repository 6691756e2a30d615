mkdir -p gpurun_out
for L in U V; do VEIL_LIB=build_ab/libveil_$L.so python tools/shard_sweep.py stack64k tiny4m mixed16m > gpurun_out/ab25_sweep_$L.log 2>&1; echo $L; grep -E "G=(1|4|8)" gpurun_out/ab25_sweep_$L.log | cut -c1-90; done
AB_WORKLOADS=stack64k,boxes1080,tiny4m python tools/ab_time.py build_ab/libveil_U.so build_ab/libveil_V.so > gpurun_out/ab25.log 2>&1; cat gpurun_out/ab25.log
python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_depth_filter.py tests/test_multi_device_gpu.py tests/test_multirank_gpu.py tests/test_checked_build_gpu.py > gpurun_out/ab25_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab25_tests.log

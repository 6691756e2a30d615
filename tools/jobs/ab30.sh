mkdir -p gpurun_out/ab30
for L in Y Z; do VEIL_LIB=build_ab/libveil_$L.so python tools/shard_sweep.py stack64k tiny4m > gpurun_out/ab30/sweep_$L.log 2>&1; echo $L; grep -E "G=(1|2|4|8)" gpurun_out/ab30/sweep_$L.log | cut -c1-200; done
AB_WORKLOADS=stack64k,boxes1080,tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_Y.so build_ab/libveil_Z.so > gpurun_out/ab30/ab.log 2>&1; cat gpurun_out/ab30/ab.log
python -m pytest -q -p no:cacheprovider tests/test_gpu_timed.py tests/test_multi_device_gpu.py > gpurun_out/ab30/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab30/tests.log

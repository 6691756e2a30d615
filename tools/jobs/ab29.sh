mkdir -p gpurun_out/ab29
for L in X Y; do VEIL_LIB=build_ab/libveil_$L.so python tools/shard_sweep.py stack64k tiny4m mixed16m > gpurun_out/ab29/sweep_$L.log 2>&1; echo $L; grep -E "G=(1|2|4|8)" gpurun_out/ab29/sweep_$L.log | cut -c1-200; done
python -m pytest -q -p no:cacheprovider tests/test_multi_device_gpu.py tests/test_multirank_gpu.py tests/test_gpu_parity.py > gpurun_out/ab29/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab29/tests.log

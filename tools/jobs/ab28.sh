mkdir -p gpurun_out/ab28
for L in U X; do
  VEIL_LIB=build_ab/libveil_$L.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab28/launch_$L.csv python tools/profile_frame.py stack64k 6 > /dev/null 2>&1; echo $L rc=$?
  VEIL_LIB=build_ab/libveil_$L.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab28/launch8_$L.csv python tools/profile_frame.py stack64k 6 0 8 > /dev/null 2>&1; echo $L rc=$?
done
for L in U X; do VEIL_LIB=build_ab/libveil_$L.so python tools/shard_sweep.py stack64k mixed16m > gpurun_out/ab28/sweep_$L.log 2>&1; echo $L; grep -E "G=(1|2|4|8)" gpurun_out/ab28/sweep_$L.log | cut -c1-90; done
AB_WORKLOADS=stack64k,boxes1080,tiny4m python tools/ab_time.py build_ab/libveil_U.so build_ab/libveil_X.so > gpurun_out/ab28/ab.log 2>&1; cat gpurun_out/ab28/ab.log
python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_multi_device_gpu.py tests/test_gpu_depth_filter.py > gpurun_out/ab28/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab28/tests.log

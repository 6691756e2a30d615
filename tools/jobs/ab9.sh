mkdir -p gpurun_out
AB_WORKLOADS=tiny4m,stack64k python tools/ab_time.py build_ab/libveil_F.so build_ab/libveil_G.so > gpurun_out/ab9.log 2>&1; cat gpurun_out/ab9.log
python tools/shard_sweep.py tiny4m > gpurun_out/sw9.log 2>&1; VEIL_LIB=$PWD/build_ab/libveil_G.so python tools/shard_sweep.py tiny4m >> gpurun_out/sw9.log 2>&1; cat gpurun_out/sw9.log

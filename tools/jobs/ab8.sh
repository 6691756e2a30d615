mkdir -p gpurun_out
AB_WORKLOADS=tiny4m,mixed16m,stack64k python tools/ab_time.py build_ab/libveil_prevF.so build_ab/libveil_F.so > gpurun_out/ab8.log 2>&1; cat gpurun_out/ab8.log

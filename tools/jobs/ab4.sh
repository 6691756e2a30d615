mkdir -p gpurun_out
AB_WORKLOADS=stack64k python tools/ab_time.py build_ab/libveil_prev.so build_ab/libveil_A.so build_ab/libveil_B.so > gpurun_out/ab4.log 2>&1; cat gpurun_out/ab4.log

mkdir -p gpurun_out/ab56
AB_WORKLOADS=tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AR.so build_ab/libveil_HACK.so > gpurun_out/ab56/ab.log 2>&1; cat gpurun_out/ab56/ab.log

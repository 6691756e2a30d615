mkdir -p gpurun_out/ab55
AB_WORKLOADS=stack64k,boxes1080,tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AR.so build_ab/libveil_AU.so > gpurun_out/ab55/ab.log 2>&1; cat gpurun_out/ab55/ab.log

mkdir -p gpurun_out/ab52
AB_WORKLOADS=stack64k,tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AR.so build_ab/libveil_AS.so > gpurun_out/ab52/ab.log 2>&1; cat gpurun_out/ab52/ab.log

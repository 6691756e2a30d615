mkdir -p gpurun_out
for i in 1 2; do AB_WORKLOADS=stack64k python tools/ab_time.py build_ab/libveil_prev.so build_ab/libveil_D.so; done > gpurun_out/ab6.log 2>&1; cat gpurun_out/ab6.log

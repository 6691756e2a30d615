mkdir -p gpurun_out
for i in 1 2; do AB_WORKLOADS=stack64k python tools/ab_time.py build_ab/libveil_prevJ.so build_ab/libveil_J.so; done > gpurun_out/ab12.log 2>&1; cat gpurun_out/ab12.log

mkdir -p gpurun_out/ab36
AB_WORKLOADS=stack64k,boxes1080 python tools/ab_time.py build_ab/libveil_AD.so build_ab/libveil_SKIP.so > gpurun_out/ab36/a.log 2>&1
VEIL_SKIP_TEST=1 AB_WORKLOADS=stack64k,boxes1080 python tools/ab_time.py build_ab/libveil_AD.so build_ab/libveil_SKIP.so > gpurun_out/ab36/b.log 2>&1
cat gpurun_out/ab36/a.log gpurun_out/ab36/b.log

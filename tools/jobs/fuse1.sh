mkdir -p gpurun_out
python -m pytest -q -p no:cacheprovider -x tests/test_gpu_fullsize.py -k c4 tests/test_gpu_parity.py -k "tiny or c4" > gpurun_out/fuse_c4.log 2>&1; echo c4 rc=$?; tail -3 gpurun_out/fuse_c4.log
VEIL_FUSED=1 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_depth_filter.py > gpurun_out/fuse_forced.log 2>&1; echo forced rc=$?; tail -15 gpurun_out/fuse_forced.log
AB_WORKLOADS=tiny4m,mixed16m,stack64k python tools/ab_time.py build_ab/libveil_base.so build_ab/libveil_lb6.so build_ab/libveil_lb5.so > gpurun_out/ab_fuse.log 2>&1; cat gpurun_out/ab_fuse.log

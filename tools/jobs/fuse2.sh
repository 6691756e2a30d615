mkdir -p gpurun_out
export AB_WORKLOADS=tiny4m,mixed16m
python tools/ab_time.py build_ab/libveil_base.so build_ab/libveil_f6.so build_ab/libveil_f5.so > gpurun_out/ab_fuse2.log 2>&1
VEIL_FUSED_READ=1 python tools/ab_time.py build_ab/libveil_f6.so > gpurun_out/ab_fuse2_read.log 2>&1
VEIL_FUSED=0 python tools/ab_time.py build_ab/libveil_f6.so > gpurun_out/ab_fuse2_off.log 2>&1
cat gpurun_out/ab_fuse2*.log
VEIL_LIB=$PWD/build_ab/libveil_f6.so timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:k_extract' --launch-skip 9 --launch-count 1 -f \
  -o gpurun_out/fx_c4 python tools/profile_frame.py tiny4m 2 > gpurun_out/ncu_fx_c4.log 2>&1; echo ncu rc=$?

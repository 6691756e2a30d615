mkdir -p gpurun_out/ab27
for L in U V; do
  VEIL_LIB=build_ab/libveil_$L.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab27/launch_$L.csv python tools/profile_frame.py stack64k 6 > /dev/null 2>&1; echo $L rc=$?
  VEIL_LIB=build_ab/libveil_$L.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab27/launch8_$L.csv python tools/profile_frame.py stack64k 6 0 8 > /dev/null 2>&1; echo $L rc=$?
done

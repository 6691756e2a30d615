mkdir -p gpurun_out/ps5
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_setup' --launch-skip 2 --launch-count 2 -f \
  -o gpurun_out/ps5/setup_c5 python tools/profile_frame.py mixed16m 2 > gpurun_out/ps5/ncu.log 2>&1; echo rc=$?

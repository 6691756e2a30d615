mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_setup' --launch-skip 2 --launch-count 2 -f \
  -o gpurun_out/setup_c4 python tools/profile_frame.py tiny4m 2 > gpurun_out/ncu_setup_c4.log 2>&1; echo rc=$?

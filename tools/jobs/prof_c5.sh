mkdir -p gpurun_out/c5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5/launch.csv python tools/profile_frame.py mixed16m 2 > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_shade' --launch-skip 2 --launch-count 2 -f \
  -o gpurun_out/c5/shade python tools/profile_frame.py mixed16m 2 > gpurun_out/c5/ncu_shade.log 2>&1; echo rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_extract' --launch-skip 6 --launch-count 1 -f \
  -o gpurun_out/c5/extract python tools/profile_frame.py mixed16m 2 > gpurun_out/c5/ncu_extract.log 2>&1; echo rc=$?

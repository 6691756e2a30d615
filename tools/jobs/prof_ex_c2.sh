mkdir -p gpurun_out/px
# frame 2's launches: k_extract low-s is the 5th k_extract (index 4)
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_extract' --launch-skip 4 --launch-count 1 -f \
  -o gpurun_out/px/extract_c2 python tools/profile_frame.py stack64k 2 > gpurun_out/px/ncu.log 2>&1; echo rc=$?
python tools/ncu_lines.py gpurun_out/px/extract_c2.ncu-rep 400 > gpurun_out/px/lines.txt 2>&1

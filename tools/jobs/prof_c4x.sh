mkdir -p gpurun_out
# frame 2's launches: k_extract low-s(4) low-g(5) high-s(6)
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_extract' --launch-skip 6 --launch-count 1 -f \
  -o gpurun_out/extract_c4 python tools/profile_frame.py tiny4m 2 > gpurun_out/ncu_extract_c4.log 2>&1; echo rc=$?
python tools/ncu_lines.py gpurun_out/extract_c4.ncu-rep 60 > gpurun_out/extract_c4_lines.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_setup_tris' --launch-skip 2 --launch-count 1 -f \
  -o gpurun_out/setup_c4 python tools/profile_frame.py tiny4m 2 > gpurun_out/ncu_setup_c4.log 2>&1; echo rc=$?
python tools/ncu_lines.py gpurun_out/setup_c4.ncu-rep 40 > gpurun_out/setup_c4_lines.txt 2>&1

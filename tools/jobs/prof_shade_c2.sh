mkdir -p gpurun_out/ps
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_shade' --launch-skip 2 --launch-count 1 -f \
  -o gpurun_out/ps/shade_c2 python tools/profile_frame.py stack64k 2 > gpurun_out/ps/ncu.log 2>&1; echo rc=$?
python tools/ncu_lines.py gpurun_out/ps/shade_c2.ncu-rep 60 > gpurun_out/ps/lines.txt 2>&1
ncu -i gpurun_out/ps/shade_c2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread > gpurun_out/ps/metrics.csv 2>/dev/null

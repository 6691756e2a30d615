mkdir -p gpurun_out
set -x
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
K='regex:k_extract|k_order_bins|k_shade|k_finalize'
for w in tiny4m mixed16m; do
  timeout 300 ncu --metrics $M --clock-control none -k "$K" --launch-skip 8 --launch-count 8 -f -o gpurun_out/${w}_raster python tools/profile_frame.py $w 2 > gpurun_out/ncu_${w}_raster.log 2>&1
  echo $w raster rc=$?
done
cp profiles/traffic.json gpurun_out/traffic.json
for w in tiny4m mixed16m; do python tools/ncu_traffic.py gpurun_out/${w}_raster.ncu-rep $w gpurun_out/traffic.json > gpurun_out/traffic_$w.log 2>&1; echo traffic $w rc=$?; done
timeout 900 ncu --set full --import-source on --clock-control none --launch-skip 15 --launch-count 15 -f -o gpurun_out/c4_frame python tools/profile_frame.py tiny4m 2 > gpurun_out/ncu_c4_frame.log 2>&1
echo c4 full rc=$?
ncu -i gpurun_out/c4_frame.ncu-rep --page details --csv > gpurun_out/c4_frame_details.csv 2>/dev/null
ncu -i gpurun_out/c4_frame.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active > gpurun_out/c4_frame_dram.csv 2>/dev/null
rm -f gpurun_out/mixed16m_raster.ncu-rep
ls -la gpurun_out

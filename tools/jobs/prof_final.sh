mkdir -p gpurun_out/pf
O=gpurun_out/pf
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_stack64k.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1; echo launches rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_tiny4m.csv \
  python bench.py --workload tiny4m --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches4.log 2>&1; echo launches4 rc=$?
K='regex:k_extract|k_order_bins|k_shade|k_finalize'
timeout 900 ncu --set full --import-source on --clock-control none -k "$K" --launch-skip 8 --launch-count 8 -f \
  -o $O/raster_stack64k python tools/profile_frame.py stack64k 2 > $O/ncu_raster_c2.log 2>&1; echo raster rc=$?
ncu -i $O/raster_stack64k.ncu-rep --page details --csv > $O/raster_stack64k_details.csv 2>/dev/null
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
ncu -i $O/raster_stack64k.ncu-rep --page raw --csv --metrics $M > $O/raster_stack64k_metrics.csv 2>/dev/null
cp profiles/traffic.json $O/traffic.json
python tools/ncu_traffic.py $O/raster_stack64k.ncu-rep stack64k $O/traffic.json > $O/traffic_stack64k.log 2>&1
python tools/ncu_lines.py $O/raster_stack64k.ncu-rep 40 -k regex:k_shade --launch-skip 0 --launch-count 1 > $O/k_shade_lines.txt 2>&1
python tools/ncu_lines.py $O/raster_stack64k.ncu-rep 30 -k regex:k_extract --launch-skip 0 --launch-count 1 > $O/k_extract_lines.txt 2>&1
rm -f $O/raster_stack64k.ncu-rep
ls -la $O

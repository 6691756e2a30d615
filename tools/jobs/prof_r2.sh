# Round-2 evidence: tests, bench lines, ncu launch list and captures.
mkdir -p gpurun_out/r2
O=gpurun_out/r2
python -m pytest -q -p no:cacheprovider tests -m gpu > $O/gputest.log 2>&1; echo "gpu tests rc=$?"; tail -3 $O/gputest.log
for w in stack64k tiny4m boxes1080 mixed16m; do
  timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; echo bench $w rc=$?
done
timeout 600 python bench.py --df 16 --no-cpu-baseline > $O/bench_stack64k_df16.json 2>&1
timeout 600 python bench.py --df 64 --no-cpu-baseline > $O/bench_stack64k_df64.json 2>&1
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_stack64k.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1; echo launches rc=$?
K='regex:k_extract|k_order_bins|k_shade|k_finalize'
timeout 900 ncu --set full --import-source on --clock-control none -k "$K" --launch-skip 8 --launch-count 8 -f \
  -o $O/raster_stack64k python tools/profile_frame.py stack64k 2 > $O/ncu_raster_c2.log 2>&1; echo raster rc=$?
ncu -i $O/raster_stack64k.ncu-rep --page details --csv > $O/raster_stack64k_details.csv 2>/dev/null
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
ncu -i $O/raster_stack64k.ncu-rep --page raw --csv --metrics $M > $O/raster_stack64k_metrics.csv 2>/dev/null
cp profiles/traffic.json $O/traffic.json
python tools/ncu_traffic.py $O/raster_stack64k.ncu-rep stack64k $O/traffic.json > $O/traffic_stack64k.log 2>&1
for w in tiny4m mixed16m; do
  timeout 600 ncu --metrics $M --clock-control none -k "$K" --launch-skip 8 --launch-count 8 -f -o $O/${w}_raster python tools/profile_frame.py $w 2 > $O/ncu_${w}_raster.log 2>&1
  python tools/ncu_traffic.py $O/${w}_raster.ncu-rep $w $O/traffic.json > $O/traffic_$w.log 2>&1
done
timeout 900 ncu --metrics $M --clock-control none --launch-skip 15 --launch-count 15 -f -o $O/c4_frame python tools/profile_frame.py tiny4m 2 > $O/ncu_c4_frame.log 2>&1; echo c4 rc=$?
ncu -i $O/c4_frame.ncu-rep --page raw --csv --metrics $M > $O/c4_kernels_dram.csv 2>/dev/null
rm -f $O/mixed16m_raster.ncu-rep $O/tiny4m_raster.ncu-rep
python tools/shard_sweep.py stack64k tiny4m mixed16m > $O/shard_sweep.log 2>&1
ls -la $O

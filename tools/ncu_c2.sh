# C2 evidence: bench lines, launch list of a short bench run, full capture of
# one frame's rasterizer kernels (+ its DRAM traffic into gpurun_out/traffic.json)
mkdir -p gpurun_out
for w in stack64k tiny4m mixed16m boxes1080; do
  timeout 300 python bench.py --workload $w > gpurun_out/bench3_$w.json 2> gpurun_out/bench3_$w.err; echo bench $w rc=$?
done
timeout 300 python bench.py --impl reference > gpurun_out/bench3_reference.json 2> gpurun_out/bench3_reference.err; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_stack64k.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1; echo launches rc=$?
K='regex:k_extract|k_order_bins|k_shade|k_finalize'
timeout 600 ncu --set full --import-source on --clock-control none -k "$K" --launch-skip 8 --launch-count 8 -f \
  -o gpurun_out/raster_stack64k python tools/profile_frame.py stack64k 2 > gpurun_out/ncu_raster_c2.log 2>&1; echo raster rc=$?
ncu -i gpurun_out/raster_stack64k.ncu-rep --page details --csv > gpurun_out/raster_stack64k_details.csv 2>/dev/null
cp profiles/traffic.json gpurun_out/traffic.json
python tools/ncu_traffic.py gpurun_out/raster_stack64k.ncu-rep stack64k gpurun_out/traffic.json > gpurun_out/traffic_stack64k.log 2>&1; echo traffic rc=$?

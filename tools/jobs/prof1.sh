mkdir -p gpurun_out
set -x
# DF 12/16 heap: shared vs global
for df in 12 16; do
  python bench.py --steps 10 --warmup 3 --df $df --no-cpu-baseline --no-e2e > gpurun_out/df${df}_smem.json 2>&1
  VEIL_HEAP_GLOBAL=1 python bench.py --steps 10 --warmup 3 --df $df --no-cpu-baseline --no-e2e > gpurun_out/df${df}_glob.json 2>&1
done
python bench.py --workload tiny4m --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
# source-level capture of C2's wave-walk shading kernel
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:k_shade' --launch-skip 2 --launch-count 1 -f \
  -o gpurun_out/shade_c2 python tools/profile_frame.py stack64k 2 > gpurun_out/ncu_shade_c2.log 2>&1; echo rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k 'regex:k_extract' --launch-skip 4 --launch-count 1 -f \
  -o gpurun_out/extract_c2 python tools/profile_frame.py stack64k 2 > gpurun_out/ncu_extract_c2.log 2>&1; echo rc=$?
ls -la gpurun_out

mkdir -p gpurun_out/ab50
for cfg in "" "VEIL_WALK_MIN_U=6" "VEIL_WALK_MIN_U=9" "VEIL_WALK_MIN_U=16" "VEIL_WALK_MIN_U=24"; do
  echo "== $cfg"; env $cfg AB_WORKLOADS=tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AQ.so 2>&1 | tail -2
done > gpurun_out/ab50/env.log 2>&1; cat gpurun_out/ab50/env.log

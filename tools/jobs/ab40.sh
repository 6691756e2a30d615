mkdir -p gpurun_out/ab40
for cfg in "" "VEIL_BULK_STAGE=0" "VEIL_WALK_MIN=4" "VEIL_WALK_MIN=9" "VEIL_NO_PDL=1"; do
  echo "== $cfg"; env $cfg AB_WORKLOADS=stack64k,boxes1080,tiny4m python tools/ab_time.py build_ab/libveil_AH.so 2>&1 | tail -3
done > gpurun_out/ab40/env.log 2>&1; cat gpurun_out/ab40/env.log

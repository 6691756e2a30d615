mkdir -p gpurun_out/ab59
for L in AV AW AV AW; do for df in 3 64; do VEIL_LIB=build_ab/libveil_$L.so timeout 300 python bench.py --df $df --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab59/b_${L}_$df.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/ab59/b_${L}_$df.json'));print('$L', $df, round(d['ms_per_step'],4), round(d['stages_ms']['shade'],4))"; done; done
AB_WORKLOADS=tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AV.so build_ab/libveil_AW.so

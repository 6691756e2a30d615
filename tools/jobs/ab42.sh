mkdir -p gpurun_out/ab42
AB_WORKLOADS=stack64k,boxes1080 python tools/ab_time.py build_ab/libveil_AH.so build_ab/libveil_EV.so > gpurun_out/ab42/a.log 2>&1
VEIL_FEW_EVENTS_TEST=1 AB_WORKLOADS=stack64k,boxes1080 python tools/ab_time.py build_ab/libveil_EV.so > gpurun_out/ab42/b.log 2>&1
cat gpurun_out/ab42/a.log gpurun_out/ab42/b.log
for L in AH EV; do VEIL_LIB=build_ab/libveil_$L.so timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab42/bench_$L.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/ab42/bench_$L.json'));print('$L', d['ms_per_step'])"; done
VEIL_FEW_EVENTS_TEST=1 VEIL_LIB=build_ab/libveil_EV.so timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab42/bench_few.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/ab42/bench_few.json'));print('few', d['ms_per_step'])"

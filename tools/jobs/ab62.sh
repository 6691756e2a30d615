mkdir -p gpurun_out/ab62
AB_WORKLOADS=stack64k,boxes1080,tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AV.so build_ab/libveil_AY.so > gpurun_out/ab62/ab.log 2>&1; cat gpurun_out/ab62/ab.log
for L in AV AY AV AY; do for w in stack64k boxes1080; do VEIL_LIB=build_ab/libveil_$L.so timeout 300 python bench.py --workload $w --steps 20 --warmup 10 --no-cpu-baseline > gpurun_out/ab62/b_${L}_$w.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/ab62/b_${L}_$w.json'));print('$L', '$w', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4))"; done; done
python -m pytest -q -x -p no:cacheprovider tests -m gpu > gpurun_out/ab62/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab62/tests.log

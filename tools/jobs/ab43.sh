mkdir -p gpurun_out/ab43
AB_WORKLOADS=stack64k,boxes1080,tiny4m,mixed16m python tools/ab_time.py build_ab/libveil_AH.so build_ab/libveil_AJ.so > gpurun_out/ab43/ab.log 2>&1; cat gpurun_out/ab43/ab.log
for L in AH AJ; do VEIL_LIB=build_ab/libveil_$L.so timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab43/bench_$L.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/ab43/bench_$L.json'));print('$L', d['ms_per_step'])"; done
python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_multi_device_gpu.py tests/test_gpu_depth_filter.py > gpurun_out/ab43/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab43/tests.log

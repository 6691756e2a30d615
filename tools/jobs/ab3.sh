mkdir -p gpurun_out
export AB_WORKLOADS=stack64k,boxes
python - <<'PY' > /dev/null
PY
AB_WORKLOADS=stack64k python tools/ab_time.py build_ab/libveil_prev.so paper_2405_13364_b200/libveil.so > gpurun_out/ab3.log 2>&1; cat gpurun_out/ab3.log
python bench.py --workload boxes1080 --no-cpu-baseline > gpurun_out/ab3_boxes.json 2>&1; VEIL_LIB=$PWD/build_ab/libveil_prev.so python bench.py --workload boxes1080 --no-cpu-baseline > gpurun_out/ab3_boxes_prev.json 2>&1
python -c "
import json
for f in ('gpurun_out/ab3_boxes_prev.json','gpurun_out/ab3_boxes.json'):
    for l in open(f):
        if l.startswith('{'): d=json.loads(l); print(f, d['ms_per_step'], d['stages_ms'])
"
python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "c2 or c3 or synthetic or golden" > gpurun_out/ab3_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab3_tests.log

mkdir -p gpurun_out
python -m pytest -q -p no:cacheprovider tests/test_gpu_depth_filter.py tests/test_gpu_fullsize.py -k "depth_filter or other_depth" > gpurun_out/ring_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/ring_tests.log
for df in 12 16 32 64; do
  python bench.py --steps 10 --warmup 3 --df $df --no-cpu-baseline --no-e2e > gpurun_out/ring_df${df}_smem.json 2>&1
  VEIL_DFM_GLOBAL=1 python bench.py --steps 10 --warmup 3 --df $df --no-cpu-baseline --no-e2e > gpurun_out/ring_df${df}_glob.json 2>&1
done
for f in gpurun_out/ring_df*.json; do python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'): d=json.loads(l); print('$f', round(d['ms_per_step'],3), round(d['stages_ms']['shade'],3))
"; done

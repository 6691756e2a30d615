mkdir -p gpurun_out/tb1
for w in stack64k boxes1080 tiny4m; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tb1/$w.json 2> gpurun_out/tb1/$w.err; echo $w rc=$?
  python -c "import json;d=json.load(open('gpurun_out/tb1/$w.json'));print('$w', d['ms_per_step'], d['stages_ms']['total'], d['e2e']['ms_per_step'])"
done
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_multirank_gpu.py > gpurun_out/tb1/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/tb1/tests.log

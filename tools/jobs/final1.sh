# full GPU suite + bench lines of every workload + smoke
mkdir -p gpurun_out/f1
O=gpurun_out/f1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
python -m pytest -q -p no:cacheprovider tests -m gpu > $O/gputest.log 2>&1; echo "gpu tests rc=$?"; tail -3 $O/gputest.log
for w in stack64k tiny4m boxes1080 mixed16m; do
  timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; echo bench $w rc=$?
done
timeout 600 python bench.py --df 16 --no-cpu-baseline > $O/bench_stack64k_df16.json 2>&1
timeout 600 python bench.py --df 64 --no-cpu-baseline > $O/bench_stack64k_df64.json 2>&1
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo ref rc=$?
timeout 600 python bench.py --impl reference --workload tiny4m --steps 3 --warmup 1 > $O/bench_reference_tiny4m.json 2>&1
python tools/shard_sweep.py stack64k tiny4m mixed16m > $O/shard_sweep.log 2>&1
for f in $O/bench_*.json; do python -c "
import json
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l)
        if 'unavailable' in d: print('$f', d['unavailable']); continue
        print('$f', round(d['ms_per_step'],3), round(d['value'],3), (d.get('e2e') or {}).get('ms_per_step'), (d.get('parity') or {}).get('identical'), d.get('stages_ms'))
"; done

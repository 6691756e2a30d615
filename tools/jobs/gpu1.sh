mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -k "not sanitizer" -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc $?"
tail -30 gpurun_out/gputest.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc $?"
python bench.py --steps 10 --warmup 3 --df 16 --no-cpu-baseline > gpurun_out/bench_c2_df16.json 2>&1
python bench.py --steps 10 --warmup 3 --df 64 --no-cpu-baseline > gpurun_out/bench_c2_df64.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -k "sanitizer" -p no:cacheprovider > gpurun_out/sanitizer.log 2>&1; echo "san rc $?"
tail -5 gpurun_out/sanitizer.log

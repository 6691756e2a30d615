mkdir -p gpurun_out
for i in 1 2; do
VEIL_WAVE1=1 python tools/quick_time.py > gpurun_out/qt_wave1_$i.log 2>&1
python tools/quick_time.py > gpurun_out/qt_wave2_$i.log 2>&1
done
python -m pytest -q -p no:cacheprovider tests/test_gpu_fullsize.py -k "c2 or c3" tests/test_gpu_parity.py > gpurun_out/ab1_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/ab1_tests.log
grep -h "stack64k ms" gpurun_out/qt_*.log

mkdir -p gpurun_out
python -m pytest -q -p no:cacheprovider tests/test_multi_device_gpu.py > gpurun_out/multi2.log 2>&1; echo rc=$?; tail -5 gpurun_out/multi2.log
VEIL_BULK_STAGE=1 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "not c4" > gpurun_out/bulk_tests.log 2>&1; echo bulk rc=$?; tail -3 gpurun_out/bulk_tests.log
export AB_WORKLOADS=stack64k,tiny4m
for i in 1 2; do
VEIL_BULK_STAGE=0 python tools/ab_time.py paper_2405_13364_b200/libveil.so > gpurun_out/bulk0_$i.log 2>&1
VEIL_BULK_STAGE=1 python tools/ab_time.py paper_2405_13364_b200/libveil.so > gpurun_out/bulk1_$i.log 2>&1
done
tail -n2 gpurun_out/bulk*_?.log
python tools/shard_sweep.py stack64k tiny4m > gpurun_out/shard_sweep.log 2>&1; cat gpurun_out/shard_sweep.log

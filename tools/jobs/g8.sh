mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --launch-skip 15 --launch-count 15 --log-file gpurun_out/g8_tiny4m.csv python tools/profile_frame.py tiny4m 2 0 8 > gpurun_out/g8.log 2>&1; echo rc=$?
AB_WORKLOADS=stack64k,tiny4m python tools/ab_time.py build_ab/libveil_D.so build_ab/libveil_E.so > gpurun_out/ab7.log 2>&1; cat gpurun_out/ab7.log
python -m pytest -q -p no:cacheprovider tests/test_gpu_abuffer_fullsize.py > gpurun_out/abuf.log 2>&1; echo abuf rc=$?; tail -15 gpurun_out/abuf.log

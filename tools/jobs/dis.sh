mkdir -p gpurun_out
python -m pytest -q -p no:cacheprovider tests/test_gpu_depth_filter.py -k "disorder or acceptance" > gpurun_out/dis.log 2>&1; echo rc=$?; tail -15 gpurun_out/dis.log

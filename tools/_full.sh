mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_device_fullsize.py -q -x --durations=6 > gpurun_out/full_test.log 2>&1; echo test=$?
tail -12 gpurun_out/full_test.log

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_geometry.py -q -x --durations=5 > gpurun_out/geo1_test.log 2>&1; echo test=$?
tail -15 gpurun_out/geo1_test.log

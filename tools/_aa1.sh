mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_single_copy.py -q -x > gpurun_out/aa1_test.log 2>&1; echo test=$?
tail -30 gpurun_out/aa1_test.log
timeout 900 python tools/kernel_sweep.py --run-env '{"two": {}, "two_nopf": {"SPLBM_L2PF": 0}, "aa": {"SPLBM_SINGLE_COPY": 1}, "aa_nopf": {"SPLBM_SINGLE_COPY": 1, "SPLBM_L2PF": 0}}' > gpurun_out/aa1_sweep.log 2>&1; echo sweep=$?
grep -v "^{" gpurun_out/aa1_sweep.log

mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_device_parity.py tests/test_device_single_copy.py -q -x > gpurun_out/pf3_test.log 2>&1; echo test=$?
tail -3 gpurun_out/pf3_test.log
timeout 1500 python tools/ab.py '{"bulk": {}, "lines": {"SPLBM_PFMODE": 1}, "lines_h64": {"SPLBM_PFMODE": 1, "SPLBM_LDHINT": 1}, "lines_pf2": {"SPLBM_PFMODE": 1, "SPLBM_L2PF": 296}, "nopf": {"SPLBM_L2PF": 0}}' --rounds 7 --steps 64 > gpurun_out/pf3_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/pf3_ab.log

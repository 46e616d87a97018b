mkdir -p gpurun_out
SPLBM_X2=1 timeout 1500 python -m pytest tests/test_device_parity.py -q -x > gpurun_out/x2d_test.log 2>&1; echo test=$?
grep -E "passed|failed" gpurun_out/x2d_test.log | tail -2
timeout 1500 python tools/ab.py '{"f64": {}, "f64_x2": {"SPLBM_X2": 1}}' channel128 ras256_phi02 full256 cavity2d_4096_a4 --rounds 9 --steps 128 > gpurun_out/x2d_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/x2d_ab.log | cut -c1-300

mkdir -p gpurun_out
SPLBM_PERSIST=1 timeout 1500 python -m pytest tests/test_device_parity.py tests/test_device_f32.py tests/test_device_golden.py -m gpu -q -x > gpurun_out/pers1_test.log 2>&1; echo test=$?
tail -3 gpurun_out/pers1_test.log
timeout 1500 python tools/ab.py '{"base": {}, "persist": {"SPLBM_PERSIST": 1}}' channel128 full256 ras256_phi05 ras256_phi02 vessel4096 cavity2d_4096_a4 --rounds 9 --steps 128 > gpurun_out/pers1_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/pers1_ab.log | cut -c1-300

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/list1_test.log 2>&1; echo test=$?
tail -3 gpurun_out/list1_test.log
SPLBM_LIST=1 timeout 1500 python -m pytest tests/test_device_parity.py tests/test_device_f32.py -m gpu -q -x > gpurun_out/list1_test_forced.log 2>&1; echo test_forced=$?
tail -3 gpurun_out/list1_test_forced.log
timeout 1500 python tools/ab.py '{"nolist": {"SPLBM_LIST": 0}, "list": {"SPLBM_LIST": 1}}' channel128 full256 ras256_phi05 ras256_phi02 vessel4096 --rounds 9 --steps 128 > gpurun_out/list1_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/list1_ab.log | cut -c1-300

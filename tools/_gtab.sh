mkdir -p gpurun_out
SPLBM_LIB=variants/lib_gtab.so timeout 900 python -m pytest tests/test_device_parity.py -q -x -k "step_bitwise" > gpurun_out/gtab_test.log 2>&1; echo test=$?
grep -E "passed|failed" gpurun_out/gtab_test.log | tail -2
timeout 1500 python tools/ab.py '{"base": {}, "gtab": {"LIB": "variants/lib_gtab.so"}}' channel128 ras256_phi02 full256 cavity2d_4096_a4 --rounds 9 --steps 128 > gpurun_out/gtab_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/gtab_ab.log | cut -c1-300

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rb1_test.log 2>&1; echo test=$?
tail -25 gpurun_out/rb1_test.log
./oracle/_ref/dropin_test | tail -3
timeout 1500 python tools/ab.py '{"old": {"LIB": "variants/lib_old.so"}, "new": {}, "new_h64": {"SPLBM_LDHINT": 1}, "aa_old": {"LIB": "variants/lib_old.so", "SPLBM_SINGLE_COPY": 1}, "aa_new": {"SPLBM_SINGLE_COPY": 1}}' --rounds 7 --steps 64 > gpurun_out/rb1_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/rb1_ab.log

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/cta3_test.log 2>&1; echo test=$?
grep -E "passed|failed" gpurun_out/cta3_test.log | tail -2
timeout 1500 python tools/ab.py '{"cur_aa": {"SPLBM_SINGLE_COPY": 1}, "aa256": {"LIB": "variants/lib_aa256.so", "SPLBM_SINGLE_COPY": 1}, "cur": {}, "all256": {"LIB": "variants/lib_all256.so"}}' channel128 ras256_phi02 full256 cavity2d_4096_a4 vessel4096 --rounds 9 --steps 128 > gpurun_out/cta3_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/cta3_ab.log | cut -c1-400

mkdir -p gpurun_out
timeout 1500 python tools/ab.py '{"f4": {"SPLBM_PRECISION": "f32"}, "f5": {"LIB": "variants/lib_f5.so", "SPLBM_PRECISION": "f32"}, "f6": {"LIB": "variants/lib_f6.so", "SPLBM_PRECISION": "f32"}, "f8": {"LIB": "variants/lib_f8.so", "SPLBM_PRECISION": "f32"}}' channel128 ras256_phi02 full256 cavity2d_4096_a4 --rounds 9 --steps 128 > gpurun_out/f32b_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/f32b_ab.log | cut -c1-400

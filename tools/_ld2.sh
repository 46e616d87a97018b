mkdir -p gpurun_out
timeout 1500 python tools/ab.py '{"prev": {"LIB": "variants/lib_prev.so"}, "cur": {}}' channel128 ras256_phi02 full256 cavity2d_4096_a4 --rounds 9 --steps 128 > gpurun_out/ld2_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/ld2_ab.log | cut -c1-300

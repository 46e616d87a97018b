mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/cta2_test.log 2>&1; echo test=$?
tail -2 gpurun_out/cta2_test.log
timeout 1500 python tools/ab.py '{"cur": {}, "s2_64": {"LIB": "variants/lib_s2_64.so"}, "s2_128": {"LIB": "variants/lib_s2_128.so"}, "s3_128": {"LIB": "variants/lib_s3_128.so"}}' channel128 ras256_phi02 cavity2d_4096_a4 vessel4096 --rounds 9 --steps 128 > gpurun_out/cta2_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/cta2_ab.log | cut -c1-400

mkdir -p gpurun_out
timeout 1500 python tools/ab.py '{"cta256": {}, "cta128": {"LIB": "variants/lib_cta128.so"}, "cta512": {"LIB": "variants/lib_cta512.so"}, "cta64": {"LIB": "variants/lib_cta64.so"}}' channel128 full256 ras256_phi05 ras256_phi02 --rounds 9 --steps 128 > gpurun_out/cta1_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/cta1_ab.log | cut -c1-400

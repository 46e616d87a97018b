timeout 1500 python tools/ab.py '{"mrt2": {"SPLBM_MODEL": "mrt"}, "mrt3": {"LIB": "variants/lib_mrt3.so", "SPLBM_MODEL": "mrt"}, "mrt4": {"LIB": "variants/lib_mrt4.so", "SPLBM_MODEL": "mrt"}}' channel128 ras256_phi02 cavity2d_4096_a4 --rounds 7 --steps 64 > gpurun_out/mrt_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/mrt_ab.log | cut -c1-300

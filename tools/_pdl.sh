mkdir -p gpurun_out
timeout 1500 python tools/ab.py '{"base": {}, "pdl_all": {"SPLBM_PDL_MIN": 0}, "nopf": {"SPLBM_L2PF": 0}, "pdl_nopf": {"SPLBM_PDL_MIN": 0, "SPLBM_L2PF": 0}}' cavity2d_256_a4 cavity2d_256_a16 --rounds 9 --steps 1024 > gpurun_out/pdl_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/pdl_ab.log | cut -c1-400

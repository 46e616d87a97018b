mkdir -p gpurun_out
timeout 1500 python tools/ab.py '{"bulk": {}, "bulk_h64": {"SPLBM_LDHINT": 1}, "nopf": {"SPLBM_L2PF": 0}, "nopf_h64": {"SPLBM_L2PF": 0, "SPLBM_LDHINT": 1}}' channel128 full256 ras256_phi05 ras256_phi02 vessel4096 --rounds 11 --steps 128 > gpurun_out/pf5_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/pf5_ab.log | cut -c1-400

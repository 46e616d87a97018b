mkdir -p gpurun_out
timeout 1500 python tools/ab.py '{"h0": {}, "h64": {"SPLBM_LDHINT": 1}, "h256": {"SPLBM_LDHINT": 2}, "h64_nopf": {"SPLBM_LDHINT": 1, "SPLBM_L2PF": 0}}' --rounds 7 --steps 64 > gpurun_out/ab3.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/ab3.log

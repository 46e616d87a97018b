mkdir -p gpurun_out
timeout 1500 python tools/ab.py '{"bulk": {}, "nopf": {"SPLBM_L2PF": 0}, "bulk2": {}, "nopf2": {"SPLBM_L2PF": 0}}' channel128 full256 ras256_phi05 ras256_phi02 --rounds 15 --steps 128 > gpurun_out/pf4_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/pf4_ab.log

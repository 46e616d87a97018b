mkdir -p gpurun_out
timeout 1500 python tools/ab.py '{"def": {}, "pf0": {"SPLBM_L2PF": 0}, "pf296": {"SPLBM_L2PF": 296}, "pf592": {"SPLBM_L2PF": 592}, "pf1184": {"SPLBM_L2PF": 1184}}' channel128 ras256_phi02 full256 cavity2d_4096_a4 vessel4096 --rounds 9 --steps 128 > gpurun_out/pf6_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/pf6_ab.log | cut -c1-500

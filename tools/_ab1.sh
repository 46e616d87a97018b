mkdir -p gpurun_out
timeout 1200 python tools/ab.py '{"pf0": {"SPLBM_L2PF": 0}, "pf148": {"SPLBM_L2PF": 148}, "pf296": {"SPLBM_L2PF": 296}, "pf592": {"SPLBM_L2PF": 592}}' --rounds 7 --steps 64 > gpurun_out/ab1.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/ab1.log

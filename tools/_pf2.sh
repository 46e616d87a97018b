mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pf2_test.log 2>&1; echo test=$?
tail -3 gpurun_out/pf2_test.log
timeout 1500 python tools/kernel_sweep.py --run-env '{"pf0": {"SPLBM_L2PF": 0}, "pf148": {"SPLBM_L2PF": 148}, "pf296": {"SPLBM_L2PF": 296}, "pf592": {"SPLBM_L2PF": 592}, "pf888": {"SPLBM_L2PF": 888}, "aa_pf296": {"SPLBM_SINGLE_COPY": 1, "SPLBM_L2PF": 296}, "aa_pf592": {"SPLBM_SINGLE_COPY": 1, "SPLBM_L2PF": 592}}' > gpurun_out/pf2_sweep.log 2>&1; echo sweep=$?
grep -v "^{" gpurun_out/pf2_sweep.log

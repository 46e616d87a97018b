mkdir -p gpurun_out
SPLBM_COMPACT=1 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/cmp1_test_forced.log 2>&1; echo test_forced=$?
grep -E "passed|failed|Error" gpurun_out/cmp1_test_forced.log | tail -5
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/cmp1_test.log 2>&1; echo test=$?
grep -E "passed|failed" gpurun_out/cmp1_test.log | tail -3
timeout 1500 python tools/ab.py '{"uniform": {"SPLBM_COMPACT": 0}, "compact": {"SPLBM_COMPACT": 1}}' channel128 ras256_phi02 ras256_phi05 full256 vessel4096 cavity2d_4096_a4 --rounds 9 --steps 128 > gpurun_out/cmp1_ab.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/cmp1_ab.log | cut -c1-300

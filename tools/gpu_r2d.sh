#!/bin/bash
# Round 2, fourth GPU session: pipelined-step parity and A/B.
mkdir -p gpurun_out/r2d
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_device_pipe.py tests/test_device_order.py -m gpu -q -x > gpurun_out/r2d/pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2d/pytest.log
timeout 1200 python tools/ab.py '{"base": {}, "pipe": {"SPLBM_PIPE": "1"}, "pipe8": {"SPLBM_PIPE": "1", "LIB": "variants/lib_pipe8.so"}}' channel128 ras256_phi02 ras256_phi05 full256 --rounds 5 --steps 64 > gpurun_out/r2d/ab_pipe.log 2>&1; echo ab=$?
tail -5 gpurun_out/r2d/ab_pipe.log
for pp in 0 1; do SPLBM_PIPE=$pp timeout 600 python tools/size_probe.py 1024 1024 1024 0.2 >> gpurun_out/r2d/size_probe.log 2>&1; done
cat gpurun_out/r2d/size_probe.log
SPLBM_PIPE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 4 -c 1 -o gpurun_out/r2d/full_pipe_ras256_phi02 python tools/profile_case.py ras256_phi02 6 > gpurun_out/r2d/ncu_pipe.log 2>&1; echo ncu=$?
ncu -i gpurun_out/r2d/full_pipe_ras256_phi02.ncu-rep --page raw --csv > gpurun_out/r2d/raw_pipe_ras256_phi02.csv 2>/dev/null

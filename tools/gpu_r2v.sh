#!/bin/bash
# Round 2: parity of the D2Q9 f64 two-nodes-per-thread step (oracle, full-size goldens, slabs).
O=gpurun_out/r2v
mkdir -p $O
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests/test_device_parity.py tests/test_device_fullsize.py tests/test_device_golden.py tests/test_device_golden_full.py tests/test_slab_gpu.py tests/test_device_physics.py tests/test_dropin_cpp.py tests/test_device_single_copy.py -q -x > $O/pytest.log 2>&1; echo pytest=$?
tail -2 $O/pytest.log
timeout 600 python tools/ab.py '{"x2": {}, "x1": {"SPLBM_X2": "0"}}' vessel4096 cavity2d_4096_a4 --rounds 9 --steps 256 > $O/ab.txt 2>&1; echo ab=$?; head -2 $O/ab.txt

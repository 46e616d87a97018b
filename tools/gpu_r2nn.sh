#!/bin/bash
# Round 2: resident kernel with 1 / 2 / 3 CTAs per SM (configs[0]).
O=gpurun_out/r2nn
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"s1": {}, "s2": {"SPLBM_RESIDENT_PER_SM": "2"}, "s3": {"SPLBM_RESIDENT_PER_SM": "3"}, "streamed": {"SPLBM_RESIDENT": "0"}}'
timeout 900 python tools/ab.py "$V" cavity2d_256_a4 cavity2d_256_a16 --rounds 7 --steps 1000 > $O/ab.txt 2>&1; echo ab=$?; head -2 $O/ab.txt
SPLBM_RESIDENT_PER_SM=2 timeout 900 python -m pytest tests/test_device_resident.py -q -x 2>&1 | tail -1

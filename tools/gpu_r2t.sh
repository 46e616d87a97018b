#!/bin/bash
# Round 2: confirm the alternating traversal on the headline (more rounds, 200-step batches).
O=gpurun_out/r2t
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"base": {}, "rev": {"SPLBM_REVERSE": "1"}}'
timeout 1500 python tools/ab.py "$V" channel128 full256 channel64 --rounds 15 --steps 192 > $O/ab.txt 2>&1; echo ab=$?
head -3 $O/ab.txt

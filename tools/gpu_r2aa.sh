#!/bin/bash
# Round 2: L2 prefetch distance for the D2Q9 f64 two-nodes-per-thread step (8 tiles per CTA).
O=gpurun_out/r2aa
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"pf2": {}, "pf1": {"SPLBM_L2PF": "148"}, "pf3": {"SPLBM_L2PF": "444"}, "pf4": {"SPLBM_L2PF": "592"}, "pf0": {"SPLBM_L2PF": "0"}}'
timeout 1500 python tools/ab.py "$V" vessel4096 cavity2d_4096_a4 --rounds 11 --steps 192 > $O/ab.txt 2>&1; echo ab=$?
head -2 $O/ab.txt

#!/bin/bash
# Round 2: two-copy L2 prefetch distance re-check (2 / 2.5 / 3 CTAs per SM ahead).
O=gpurun_out/r2qq
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"pf2": {}, "pf25": {"SPLBM_L2PF": "370"}, "pf3": {"SPLBM_L2PF": "444"}, "pf15": {"SPLBM_L2PF": "222"}}'
timeout 1200 python tools/ab.py "$V" channel128 ras256_phi02 ras256_phi05 full256 --rounds 11 --steps 192 > $O/ab.txt 2>&1; echo ab=$?; head -4 $O/ab.txt

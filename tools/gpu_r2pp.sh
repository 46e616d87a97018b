#!/bin/bash
# Round 2: single-copy L2 prefetch distance after the phase-1 register change (16 CTAs/SM).
O=gpurun_out/r2pp
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"pf4": {"SPLBM_SINGLE_COPY": "1"}, "pf5": {"SPLBM_SINGLE_COPY": "1", "SPLBM_L2PF": "740"}, "pf6": {"SPLBM_SINGLE_COPY": "1", "SPLBM_L2PF": "888"}, "pf8": {"SPLBM_SINGLE_COPY": "1", "SPLBM_L2PF": "1184"}}'
timeout 1200 python tools/ab.py "$V" channel128 ras256_phi02 ras256_phi05 full256 --rounds 11 --steps 192 > $O/ab.txt 2>&1; echo ab=$?; head -4 $O/ab.txt

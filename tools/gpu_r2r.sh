#!/bin/bash
# Round 2: 2D (D2Q9) step tuning on the vessel tree / dense 4096^2: CTA size, register budget,
# L2 prefetch distance (interleaved A/B).
O=gpurun_out/r2r
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"base": {}, "pf1": {"SPLBM_L2PF": "148"}, "pf3": {"SPLBM_L2PF": "444"}, "pf4": {"SPLBM_L2PF": "592"}, "t128": {"LIB": "variants/lib_t2_128.so"}, "t32": {"LIB": "variants/lib_t2_32.so"}, "minb8": {"LIB": "variants/lib_minb2_8.so"}}'
timeout 1200 python tools/ab.py "$V" vessel4096 cavity2d_4096_a4 --rounds 7 --steps 64 > $O/ab.txt 2>&1; echo ab=$?
head -3 $O/ab.txt

#!/bin/bash
# Round 2: 3D step with 128-thread CTAs (two 4^3 tiles) vs 64 (one tile), interleaved A/B.
O=gpurun_out/r2ff
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"t64": {}, "t128": {"LIB": "variants/lib_t128.so"}}'
timeout 1500 python tools/ab.py "$V" channel128 ras256_phi02 ras256_phi05 full256 --rounds 11 --steps 192 > $O/ab.txt 2>&1; echo ab=$?
head -4 $O/ab.txt

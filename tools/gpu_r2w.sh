#!/bin/bash
# Round 2: two-copy 3D step with the store address re-derived after the collision (no spills at
# 64 registers; 56 registers = 18 CTAs/SM), interleaved A/B.
O=gpurun_out/r2w
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"base": {}, "rec": {"LIB": "variants/lib_rec.so"}}'
timeout 1500 python tools/ab.py "$V" channel128 ras256_phi02 ras256_phi05 full256 --rounds 15 --steps 192 > $O/ab.txt 2>&1; echo ab=$?
head -4 $O/ab.txt

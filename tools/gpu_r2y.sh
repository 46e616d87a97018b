#!/bin/bash
# Round 2: 3D MRT step at 10 CTAs/SM (94 registers, no spills) vs 12 (80 registers, 144 B spills).
O=gpurun_out/r2y
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"m12": {"SPLBM_MODEL": "mrt"}, "m10": {"SPLBM_MODEL": "mrt", "LIB": "variants/lib_mrt10.so"}}'
timeout 1500 python tools/ab.py "$V" channel128 ras256_phi05 full256 --rounds 11 --steps 128 > $O/ab.txt 2>&1; echo ab=$?
head -3 $O/ab.txt

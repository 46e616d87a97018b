#!/bin/bash
# Round 2: f32 two-node step with 128-thread CTAs vs 64.
O=gpurun_out/r2tt
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"x64": {"SPLBM_PRECISION": "f32"}, "x128": {"SPLBM_PRECISION": "f32", "LIB": "variants/lib_x2t128.so"}}'
timeout 1200 python tools/ab.py "$V" channel128 ras256_phi02 ras256_phi05 full256 --rounds 11 --steps 192 > $O/ab.txt 2>&1; echo ab=$?; head -4 $O/ab.txt

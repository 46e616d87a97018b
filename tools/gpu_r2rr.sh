#!/bin/bash
# Round 2: single-copy kernels with 128-thread CTAs (two 4^3 tiles) vs 64.
O=gpurun_out/r2rr
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"aa64": {"SPLBM_SINGLE_COPY": "1"}, "aa128": {"SPLBM_SINGLE_COPY": "1", "LIB": "variants/lib_aa128.so"}}'
timeout 1200 python tools/ab.py "$V" channel128 ras256_phi02 ras256_phi05 full256 --rounds 11 --steps 192 > $O/ab.txt 2>&1; echo ab=$?; head -4 $O/ab.txt

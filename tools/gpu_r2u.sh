#!/bin/bash
# Round 2: two nodes per thread for the D2Q9 f64 step (x2 kernel), 64- and 128-thread CTAs.
O=gpurun_out/r2u
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"base": {}, "x2": {"LIB": "variants/lib_x2f64.so"}, "x2_128": {"LIB": "variants/lib_x2f64_128.so"}}'
timeout 1500 python tools/ab.py "$V" vessel4096 cavity2d_4096_a4 --rounds 11 --steps 256 > $O/ab.txt 2>&1; echo ab=$?
head -2 $O/ab.txt

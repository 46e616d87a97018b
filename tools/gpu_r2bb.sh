#!/bin/bash
# Round 2 experiment: MRT with products shared between rows of equal K_ij (generated for tau 0.8).
O=gpurun_out/r2bb
mkdir -p $O
cd "$(dirname "$0")/.."
timeout 600 python tools/mrt_gen_check.py variants/lib_gen10.so variants/lib_gen8.so > $O/check.txt 2>&1; echo check=$?; cat $O/check.txt
V='{"aot": {"SPLBM_MODEL": "mrt"}, "gen10": {"SPLBM_MODEL": "mrt", "LIB": "variants/lib_gen10.so"}, "gen8": {"SPLBM_MODEL": "mrt", "LIB": "variants/lib_gen8.so"}}'
timeout 1500 python tools/ab.py "$V" channel128 ras256_phi05 full256 --rounds 11 --steps 128 > $O/ab.txt 2>&1; echo ab=$?
head -3 $O/ab.txt

# Round 2: single-copy phase 1 with re-derived scatter addresses (64 registers, no spills) — A/B.
mkdir -p gpurun_out
V='{"base": {"SPLBM_SINGLE_COPY": "1"}, "m3_rc": {"SPLBM_SINGLE_COPY": "1", "LIB": "variants/lib_aa1_m3_rc.so"}, "m4_rc": {"SPLBM_SINGLE_COPY": "1", "LIB": "variants/lib_aa1_m4_rc.so"}}'
timeout 900 python tools/ab.py "$V" channel128 ras256_phi02 ras256_phi05 cavity2d_4096_a4 --rounds 5 --steps 64 > gpurun_out/ab_aa1.txt 2>&1; echo ab=$?; head -4 gpurun_out/ab_aa1.txt

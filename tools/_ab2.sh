mkdir -p gpurun_out
timeout 1200 python tools/ab.py '{"two": {}, "aa": {"SPLBM_SINGLE_COPY": 1}, "aa_minb3": {"SPLBM_SINGLE_COPY": 1, "SPLBM_MINB": 3}}' channel128 ras256_phi02 full256 --rounds 7 --steps 64 > gpurun_out/ab2.log 2>&1; echo ab=$?
grep -v "^{" gpurun_out/ab2.log

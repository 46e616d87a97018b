# Round 2: resident multi-step kernel (small domains) — parity, equivalence, A/B timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_resident.py tests/test_device_parity.py -q -x > gpurun_out/resident_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/resident_tests.log
timeout 600 python tools/ab.py '{"resident": {"SPLBM_RESIDENT": "1"}, "streamed": {"SPLBM_RESIDENT": "0"}}' cavity2d_256_a4 cavity2d_256_a16 --rounds 5 --steps 1000 > gpurun_out/ab_resident.txt 2>&1; echo ab=$?; cat gpurun_out/ab_resident.txt

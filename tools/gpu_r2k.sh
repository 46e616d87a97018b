# Round 2: resident kernel — A/B and one ncu --set full capture of a 200-step configs[0] launch.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_device_resident.py -q -x > gpurun_out/resident_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/resident_tests.log
timeout 600 python tools/ab.py '{"resident": {"SPLBM_RESIDENT": "1"}, "streamed": {"SPLBM_RESIDENT": "0"}}' cavity2d_256_a4 cavity2d_256_a16 --rounds 5 --steps 1000 > gpurun_out/ab_resident.txt 2>&1; echo ab=$?; head -2 gpurun_out/ab_resident.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:resident -c 1 -o gpurun_out/ncu_resident -f python tools/profile_case.py cavity2d_256_a4 200 > gpurun_out/ncu_resident.log 2>&1; echo ncu=$?

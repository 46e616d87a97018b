mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/f32a_test.log 2>&1; echo test=$?
tail -30 gpurun_out/f32a_test.log
./oracle/_ref/dropin_test | tail -20

mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/ab1_test.log 2>&1; echo test=$?
tail -2 gpurun_out/ab1_test.log
timeout 1200 python tools/kernel_sweep.py --run > gpurun_out/ab1_sweep.log 2>&1; echo sweep=$?
timeout 1200 python tools/kernel_sweep.py --run > gpurun_out/ab1_sweep2.log 2>&1; echo sweep=$?
grep -v "^{" gpurun_out/ab1_sweep.log gpurun_out/ab1_sweep2.log

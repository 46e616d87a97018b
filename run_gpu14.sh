timeout 900 python tools/kernel_sweep.py --run > gpurun_out/sweep14.log 2>&1; echo sweep=$?
timeout 900 python tools/kernel_sweep.py --run > gpurun_out/sweep14b.log 2>&1; echo sweep=$?

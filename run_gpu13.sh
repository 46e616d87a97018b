timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu13.log 2>&1; echo pytest=$?
timeout 900 python tools/kernel_sweep.py --run > gpurun_out/sweep13.log 2>&1; echo sweep=$?

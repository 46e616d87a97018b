timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu12.log 2>&1; echo pytest=$?

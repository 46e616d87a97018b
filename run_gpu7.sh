timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu7.log 2>&1; echo pytest=$?
timeout 600 python bench.py --no-cpu > gpurun_out/bench7.log 2>&1; echo bench=$?

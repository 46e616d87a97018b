timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu16.log 2>&1; echo pytest=$?
timeout 900 python bench.py --no-cpu --no-sweep > gpurun_out/bench16.log 2>&1; echo bench=$?

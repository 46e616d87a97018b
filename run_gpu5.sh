timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu5.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench5.log 2>&1; echo bench=$?

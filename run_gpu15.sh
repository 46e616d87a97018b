timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu15.log 2>&1; echo pytest=$?
timeout 900 python bench.py --no-cpu > gpurun_out/bench15.log 2>&1; echo bench=$?

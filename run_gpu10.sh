free -g | head -2; nproc
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu10.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config ras1024 --phi 0.2 --steps 20 --warmup 3 > gpurun_out/bench10_big.log 2>&1; echo big=$?

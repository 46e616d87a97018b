timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke4.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench4.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench4_ref.log 2>&1; echo benchref=$?
timeout 900 python tools/kernel_sweep.py --run > gpurun_out/sweep4.log 2>&1; echo sweep=$?

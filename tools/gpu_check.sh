#!/bin/bash
# One gpurun call: smoke, the GPU parity suite, the default bench line. Logs under gpurun_out/.
tag=${1:-check}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo bench=$?
tail -3 gpurun_out/pytest_gpu_$tag.log

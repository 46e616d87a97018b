# Round 2: single-copy parity after the phase-1 scatter change; resident + whole GPU suite.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r2m.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu_r2m.log

timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo pytest=$?
timeout 900 python tools/kernel_sweep.py --run > gpurun_out/sweep2.log 2>&1; echo sweep=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 5 -c 1 -o gpurun_out/prof_step2 python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_full2.log 2>&1; echo ncu2=$?

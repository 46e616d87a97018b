set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Flags" | cut -c1-200
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 5 -c 1 -o gpurun_out/prof_step python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?

timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu3.log 2>&1; echo pytest=$?
timeout 900 python tools/kernel_sweep.py --run > gpurun_out/sweep3.log 2>&1; echo sweep=$?
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench3.log 2>&1; echo bench=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches3.csv python bench.py --steps 20 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1; echo ncu1=$?
for c in channel128 ras256_phi05 ras256_phi02 cavity2d_4096_a4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 3 -c 1 -o gpurun_out/prof3_$c python tools/profile_case.py $c 5 > gpurun_out/ncu3_$c.log 2>&1; echo ncu_$c=$?
done

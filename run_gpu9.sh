timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu9.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench9.log 2>&1; echo bench=$?
for c in channel128 ras256_phi02 cavity2d_4096_a4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 3 -c 1 -o gpurun_out/prof9_$c python tools/profile_case.py $c 5 > gpurun_out/ncu9_$c.log 2>&1; echo ncu_$c=$?
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches9.csv python bench.py --steps 50 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1; echo ncu_launch=$?

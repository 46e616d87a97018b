mkdir -p gpurun_out
for c in ras256_phi02 channel128; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 3 -c 1 -o gpurun_out/p2_$c python tools/profile_case.py $c 5 > gpurun_out/p2_$c.log 2>&1; echo ncu_$c=$?
done

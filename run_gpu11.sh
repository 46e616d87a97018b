timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu11.log 2>&1; echo pytest=$?
for c in ras48_periodic channel3d_small cavity2d_64_a16 random_a3; do
  for t in memcheck racecheck initcheck; do
    timeout 600 compute-sanitizer --tool $t --error-exitcode 9 python tools/profile_case.py $c 3 > gpurun_out/san_${t}_$c.log 2>&1; echo san_${t}_$c=$?
  done
done

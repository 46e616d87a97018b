mkdir -p gpurun_out
free -g | head -2
timeout 900 python -m pytest tests/test_device_single_copy.py -q -x > gpurun_out/big1_test.log 2>&1; echo test=$?; tail -2 gpurun_out/big1_test.log
for phi in 0.5 0.8; do
timeout 900 python bench.py --config ras1024 --phi $phi --single-copy --steps 20 --warmup 4 > gpurun_out/big1_aa_$phi.log 2>&1; echo big=$?
tail -c 1500 gpurun_out/big1_aa_$phi.log
done
timeout 900 python bench.py --config ras1024 --phi 0.2 --steps 20 --warmup 4 > gpurun_out/big1_two_0.2.log 2>&1; echo big=$?
tail -c 1200 gpurun_out/big1_two_0.2.log

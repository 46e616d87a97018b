#!/bin/bash
# Round 2, third GPU session: row-band traversal order at large x-y planes; order/AA parity tests.
mkdir -p gpurun_out/r2c
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_device_order.py tests/test_slab_gpu.py -m gpu -q -x > gpurun_out/r2c/pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r2c/pytest.log
for o in 0 8 16 32 64 16x64 32x128; do
  SPLBM_ORDER=$o timeout 600 python tools/size_probe.py 1024 1024 256 0.2 >> gpurun_out/r2c/size_probe.log 2>&1
done
for o in 0 16 32; do
  SPLBM_ORDER=$o timeout 600 python tools/size_probe.py 1024 1024 1024 0.2 >> gpurun_out/r2c/size_probe.log 2>&1
done
cat gpurun_out/r2c/size_probe.log
for o in 0 16; do
  SPLBM_ORDER=$o timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:t2c_step -s 4 -c 1 --csv python tools/size_probe.py 1024 1024 256 0.2 --steps 2 --warmup 4 2>&1 | grep -E "t2c_step" | cut -d, -f13- >> gpurun_out/r2c/size_ncu.log
done
cat gpurun_out/r2c/size_ncu.log

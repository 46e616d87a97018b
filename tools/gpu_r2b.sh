#!/bin/bash
# Round 2, second GPU session: full parity suite; L2-reuse (plane size) hypothesis and the column
# traversal order at 1024^3; FMA / order A/B on 256^3.
mkdir -p gpurun_out/r2b
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2b/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/r2b/pytest_gpu.log
for o in 0 32; do
  for d in "1024 1024 256" "256 256 1024" "512 512 512" "1024 1024 1024"; do
    SPLBM_ORDER=$o timeout 600 python tools/size_probe.py $d 0.2 >> gpurun_out/r2b/size_probe.log 2>&1
  done
done
for o in 16 64; do SPLBM_ORDER=$o timeout 600 python tools/size_probe.py 1024 1024 1024 0.2 >> gpurun_out/r2b/size_probe.log 2>&1; done
for o in 0 32; do SPLBM_ORDER=$o timeout 600 python tools/size_probe.py 1024 1024 1024 0.5 --single-copy >> gpurun_out/r2b/size_probe.log 2>&1; done
for o in 0 32; do SPLBM_ORDER=$o timeout 600 python tools/size_probe.py 1024 1024 1024 0.2 >> gpurun_out/r2b/size_probe.log 2>&1; done
cat gpurun_out/r2b/size_probe.log
for o in 0 32; do
  for d in "1024 1024 256" "256 256 1024"; do
    SPLBM_ORDER=$o timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:t2c_step -s 4 -c 1 --csv python tools/size_probe.py $d 0.2 --steps 2 --warmup 4 2>&1 | grep -E "t2c_step|dims" >> gpurun_out/r2b/size_ncu.log
  done
done
cat gpurun_out/r2b/size_ncu.log | cut -c1-400
timeout 900 python tools/ab.py '{"o0": {"SPLBM_ORDER": "0"}, "o16": {"SPLBM_ORDER": "16"}, "o32": {"SPLBM_ORDER": "32"}}' ras256_phi02 ras256_phi05 full256 --rounds 5 --steps 64 > gpurun_out/r2b/ab_order256.log 2>&1; echo ab=$?
tail -4 gpurun_out/r2b/ab_order256.log

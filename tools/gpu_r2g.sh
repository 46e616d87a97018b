#!/bin/bash
# Round 2: why is configs[4] (1024^3) slower per node than 256^3? ncu says the 1024^3 step reads
# 1.77x the algorithmic bytes vs 1.64x at 256^3 (a tile plane, ~200 MB, exceeds L2, so -z / +z
# face gathers miss). Traversal orders (SPLBM_ORDER=BY[xBX], row bands / columns) re-measured with
# DRAM bytes, interleaved to cancel power-cap drift.
O=gpurun_out/r2g
mkdir -p $O
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for o in 0 8 16 32 64 32x32 64x64 16x256; do
    SPLBM_ORDER=$o timeout 600 python tools/size_probe.py 1024 1024 1024 0.2 >> $O/size_probe.log 2>> $O/size_probe.err
  done
done
cat $O/size_probe.log
for o in 0 16 64 32x32; do
  SPLBM_ORDER=$o timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum \
    --replay-mode application --clock-control none --cache-control none -k regex:t2c_step -s 6 -c 1 --csv \
    python tools/size_probe.py 1024 1024 1024 0.2 --steps 2 --warmup 6 > $O/ncu_order_$o.csv 2>&1; echo ncu_$o=$?
done
for o in 0 16; do
  SPLBM_ORDER=$o timeout 600 python tools/size_probe.py 512 512 512 0.2 >> $O/size_probe512.log 2>> $O/size_probe.err
  SPLBM_ORDER=$o timeout 600 python tools/size_probe.py 512 512 512 0.2 >> $O/size_probe512.log 2>> $O/size_probe.err
done
cat $O/size_probe512.log

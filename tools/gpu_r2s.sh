#!/bin/bash
# Round 2: alternating traversal direction (SPLBM_REVERSE=1: every other step descends, starting
# on the tiles the previous step wrote last) with evict-first (.cs) or plain PDF stores; A/B +
# DRAM bytes of a descending step.
O=gpurun_out/r2s
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"base": {}, "rev": {"SPLBM_REVERSE": "1"}, "plain": {"LIB": "variants/lib_plainst.so"}, "rev_plain": {"SPLBM_REVERSE": "1", "LIB": "variants/lib_plainst.so"}}'
timeout 1500 python tools/ab.py "$V" channel128 ras256_phi02 ras256_phi05 full256 cavity2d_4096_a4 vessel4096 --rounds 7 --steps 64 > $O/ab.txt 2>&1; echo ab=$?
head -6 $O/ab.txt
for v in 0 1; do
  SPLBM_REVERSE=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --replay-mode application --cache-control none --clock-control none -k regex:t2c_step -s 5 -c 2 --csv python tools/profile_case.py channel128 8 > $O/ncu_rev$v.csv 2>&1; echo ncu$v=$?
done
grep -h "dram__bytes\|duration\|hit_rate" $O/ncu_rev*.csv | awk -F'","' '{print $1, $(NF-2), $NF}' | cut -c1-200

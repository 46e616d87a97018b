#!/bin/bash
# Round 2: L2 prefetch of only the non-solid z-layer range (SPLBM_PF_RANGE=1) vs whole blocks,
# with prefetch distances 2/3/4 CTAs per SM ahead; interleaved A/B + DRAM bytes (ncu).
O=gpurun_out/r2p
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"block2": {}, "range2": {"SPLBM_PF_RANGE": "1"}, "range3": {"SPLBM_PF_RANGE": "1", "SPLBM_L2PF": "444"}, "range4": {"SPLBM_PF_RANGE": "1", "SPLBM_L2PF": "592"}, "block3": {"SPLBM_L2PF": "444"}}'
timeout 1200 python tools/ab.py "$V" ras256_phi02 ras256_phi05 channel128 full256 --rounds 7 --steps 64 > $O/ab.txt 2>&1; echo ab=$?
cat $O/ab.txt | head -5
for v in 0 1; do
  SPLBM_PF_RANGE=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:t2c_step -s 4 -c 1 --csv python tools/profile_case.py ras256_phi02 6 > $O/ncu_range$v.csv 2>&1; echo ncu$v=$?
done
grep -h "dram__bytes\|duration" $O/ncu_range*.csv | cut -c1-300

#!/bin/bash
# Round 2: full ncu capture of the sparse step (RAS 256^3 phi 0.2) for a memory-hierarchy breakdown.
O=gpurun_out/r2q
mkdir -p $O
cd "$(dirname "$0")/.."
for c in ras256_phi02 channel128; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 4 -c 1 -o $O/full_$c python tools/profile_case.py $c 6 > $O/ncu_$c.log 2>&1; echo ncu=$?
ncu -i $O/full_$c.ncu-rep --page raw --csv > $O/raw_$c.csv 2>/dev/null
ncu -i $O/full_$c.ncu-rep --page details --csv > $O/details_$c.csv 2>/dev/null
done

#!/bin/bash
# Round 2: ncu of the final single-copy pair (128-thread CTAs) and resident configs[0] batch.
O=gpurun_out/r2uu
mkdir -p $O
cd "$(dirname "$0")/.."
ncu_full() {  # name case kregex skip count [env...]
  local n=$1 c=$2 k=$3 s=$4 cnt=$5; shift 5
  env "$@" timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $cnt \
    -o $O/full_$n python tools/profile_case.py $c ${STEPS:-6} > $O/ncu_$n.log 2>&1; echo ncu_$n=$?
  ncu -i $O/full_$n.ncu-rep --page raw --csv > $O/raw_$n.csv 2>/dev/null
  rm -f $O/full_$n.ncu-rep
}
ncu_full channel128_aa channel128 t2c_aa 4 2 SPLBM_SINGLE_COPY=1
STEPS=200 ncu_full cavity2d_256_resident cavity2d_256_a4 resident 0 1

#!/bin/bash
# Round 2 (third session), final evidence of the round-2 code: default bench + reference arm, the
# bench launch list, ncu --set full of the single-copy pair (phase-1 register diet) and of the
# resident multi-step kernel (configs[0]) exported to CSV.
O=gpurun_out/r2n
mkdir -p $O
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo benchref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 4 --warmup 3 --no-sweep --no-cpu --no-other --no-configs4 > $O/launches_bench.log 2>&1; echo launches=$?
ncu_full() {  # name case kregex skip count [env...]
  local n=$1 c=$2 k=$3 s=$4 cnt=$5; shift 5
  env "$@" timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $cnt \
    -o $O/full_$n python tools/profile_case.py $c ${STEPS:-6} > $O/ncu_$n.log 2>&1; echo ncu_$n=$?
  ncu -i $O/full_$n.ncu-rep --page raw --csv > $O/raw_$n.csv 2>/dev/null
  ncu -i $O/full_$n.ncu-rep --page details --csv > $O/details_$n.csv 2>/dev/null
  ncu -i $O/full_$n.ncu-rep --page source --csv --print-source sass > $O/source_$n.csv 2>/dev/null
  rm -f $O/full_$n.ncu-rep
}
ncu_full channel128_aa channel128 t2c_aa 4 2 SPLBM_SINGLE_COPY=1
STEPS=200 ncu_full cavity2d_256_resident cavity2d_256_a4 resident 0 1
ncu_full cavity2d_256_streamed cavity2d_256_a4 t2c_step 4 1 SPLBM_RESIDENT=0
du -sh $O

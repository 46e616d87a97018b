#!/bin/bash
# Round 2 (third session), final evidence after the register changes (two-copy step store
# re-derivation, D2Q9 f64 two nodes per thread, MRT at 10 CTAs/SM): default bench + reference
# arm, the bench launch list, ncu --set full of every step kernel the bench reports (CSV exports).
O=gpurun_out/r2n2
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
  rm -f $O/full_$n.ncu-rep
}
ncu_full channel128 channel128 t2c_step 4 1
ncu_full ras256_phi02 ras256_phi02 t2c_step 4 1
ncu_full ras256_phi05 ras256_phi05 t2c_step 4 1
ncu_full vessel4096 vessel4096_a4 t2c_step 4 1
ncu_full cavity2d_4096 cavity2d_4096_a4 t2c_step 4 1
ncu_full channel128_mrt channel128 t2c_step 4 1 SPLBM_MODEL=mrt
ncu_full channel128_f32 channel128 t2c_step 4 1 SPLBM_PRECISION=f32
du -sh $O

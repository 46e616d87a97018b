#!/bin/bash
# Round 2 (re-entry), second GPU session: default bench + reference arm (full JSON kept), launch
# list, ncu --set full of the headline / sparse / 1024^3 step exported to CSV (reports deleted:
# gpurun_out must stay under 64 MiB), TMA granularity probe, 1024^3 RN vs FMA, full GPU suite.
O=gpurun_out/r2f
mkdir -p $O
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
tail -c 300 $O/bench.json
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo benchref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 4 --warmup 3 --no-sweep --no-cpu --no-other --no-configs4 > $O/launches_bench.log 2>&1; echo launches=$?
ncu_full() {  # name case [env...]
  local n=$1 c=$2; shift 2
  env "$@" timeout 1500 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 4 -c 1 \
    -o $O/full_$n python tools/profile_case.py $c 6 > $O/ncu_$n.log 2>&1; echo ncu_$n=$?
  ncu -i $O/full_$n.ncu-rep --page raw --csv > $O/raw_$n.csv 2>/dev/null
  ncu -i $O/full_$n.ncu-rep --page details --csv > $O/details_$n.csv 2>/dev/null
  ncu -i $O/full_$n.ncu-rep --page source --csv --print-source sass > $O/source_$n.csv 2>/dev/null
  rm -f $O/full_$n.ncu-rep
}
ncu_full channel128 channel128
ncu_full ras256_phi02 ras256_phi02
ncu_full ras256_phi05 ras256_phi05
ncu_full vessel4096 vessel4096_a4
# configs[4] steady state (application replay: no save/restore of a 107 GB working set)
timeout 1500 ncu --set full --replay-mode application --clock-control none --cache-control none --import-source on \
  -k regex:t2c_step -s 4 -c 1 -o $O/full_ras1024_phi02 python tools/profile_case.py ras1024_phi02 6 > $O/ncu_ras1024_phi02.log 2>&1; echo ncu1024=$?
ncu -i $O/full_ras1024_phi02.ncu-rep --page raw --csv > $O/raw_ras1024_phi02.csv 2>/dev/null
ncu -i $O/full_ras1024_phi02.ncu-rep --page details --csv > $O/details_ras1024_phi02.csv 2>/dev/null
rm -f $O/full_ras1024_phi02.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --cache-control all --csv --log-file $O/tma_probe.csv ./tools/tma_probe > $O/tma_probe.log 2>&1; echo tmaprobe=$?
for v in rn fma rn; do
  if [ $v = fma ]; then L=paper_1703_08015_b200/libsplbm_b200_fma.so; else L=; fi
  SPLBM_LIB=$L timeout 900 python bench.py --config ras1024 --phi 0.2 --steps 20 --warmup 4 >> $O/ras1024_rn_fma.json 2>> $O/ras1024.err; echo big_$v=$?
done
timeout 2700 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 $O/pytest_gpu.log
du -sh $O

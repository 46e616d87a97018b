#!/bin/bash
# (historical: SPLBM_PIPE selected the software-pipelined step kernel, removed after this A/B)
# Round 2 (re-entry), first GPU session: smoke, default bench (N=1 line incl. configs4), reference
# arm, pipelined-step / FMA A/B, launch list + ncu --set full captures of the headline, the sparse
# RAS 256^3 phi 0.2 and the 1024^3 step.
mkdir -p gpurun_out/r2e
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2e/smoke.log 2>&1; echo smoke=$?
tail -2 gpurun_out/r2e/smoke.log
timeout 900 python bench.py > gpurun_out/r2e/bench.json.log 2>&1; echo bench=$?
tail -c 400 gpurun_out/r2e/bench.json.log
timeout 600 python bench.py --impl reference > gpurun_out/r2e/bench_ref.json.log 2>&1; echo benchref=$?
tail -c 400 gpurun_out/r2e/bench_ref.json.log
timeout 1200 python tools/ab.py '{"base": {}, "pipe": {"SPLBM_PIPE": "1"}, "pipe8": {"SPLBM_PIPE": "1", "LIB": "variants/lib_pipe8.so"}, "pipe12": {"SPLBM_PIPE": "1", "LIB": "variants/lib_pipe12.so"}, "fma": {"LIB": "paper_1703_08015_b200/libsplbm_b200_fma.so"}}' channel128 ras256_phi02 ras256_phi05 full256 --rounds 5 --steps 64 > gpurun_out/r2e/ab_pipe_fma.log 2>&1; echo ab=$?
tail -8 gpurun_out/r2e/ab_pipe_fma.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2e/launches.csv python bench.py --steps 4 --warmup 3 --no-sweep --no-cpu --no-other --no-configs4 > gpurun_out/r2e/launches_bench.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 4 -c 1 -o gpurun_out/r2e/full_channel128 python tools/profile_case.py channel128 6 > gpurun_out/r2e/ncu_ch.log 2>&1; echo ncuch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 4 -c 1 -o gpurun_out/r2e/full_ras256_phi02 python tools/profile_case.py ras256_phi02 6 > gpurun_out/r2e/ncu_ras256.log 2>&1; echo ncu256=$?
SPLBM_PIPE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 4 -c 1 -o gpurun_out/r2e/full_pipe_ras256_phi02 python tools/profile_case.py ras256_phi02 6 > gpurun_out/r2e/ncu_pipe.log 2>&1; echo ncupipe=$?
timeout 1500 ncu --set full --replay-mode application --clock-control none --cache-control none --import-source on -k regex:t2c_step -s 4 -c 1 -o gpurun_out/r2e/full_ras1024_phi02 python tools/profile_case.py ras1024_phi02 6 > gpurun_out/r2e/ncu_ras1024.log 2>&1; echo ncu1024=$?
for c in channel128 ras256_phi02 pipe_ras256_phi02 ras1024_phi02; do
  ncu -i gpurun_out/r2e/full_$c.ncu-rep --page raw --csv > gpurun_out/r2e/raw_$c.csv 2>/dev/null
done
ls -la gpurun_out/r2e

#!/bin/bash
# One gpurun call that regenerates the evidence under profiles/ (copied out of gpurun_out/ here):
# GPU parity suite, the default bench line, the reference arm, the ncu launch list of the bench
# command, one `ncu --set full` capture of the step kernel per workload, the 1024^3 lines.
mkdir -p gpurun_out/prof
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/prof/pytest_gpu.log 2>&1; echo pytest=$?
timeout 1200 python bench.py > gpurun_out/prof/bench.json.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/prof/bench_ref.json.log 2>&1; echo benchref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 50 --warmup 3 --no-sweep --no-cpu --no-other > /dev/null 2>&1; echo ncu_launch=$?
for c in channel128 ras256_phi02 ras256_phi05 cavity2d_4096_a4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 3 -c 1 -o gpurun_out/prof/full_$c python tools/profile_case.py $c 5 > gpurun_out/prof/ncu_$c.log 2>&1; echo ncu_$c=$?
done
# secondary kernels: f32 (two nodes per thread), MRT, the single-copy pair (phase 1 = launch 4, phase 2 = launch 5)
SPLBM_PRECISION=f32 timeout 600 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 3 -c 1 -o gpurun_out/prof/full_channel128_f32 python tools/profile_case.py channel128 5 > gpurun_out/prof/ncu_f32.log 2>&1; echo ncu_f32=$?
SPLBM_MODEL=mrt timeout 600 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 3 -c 1 -o gpurun_out/prof/full_channel128_mrt python tools/profile_case.py channel128 5 > gpurun_out/prof/ncu_mrt.log 2>&1; echo ncu_mrt=$?
SPLBM_SINGLE_COPY=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:t2c_aa -s 4 -c 2 -o gpurun_out/prof/full_channel128_aa python tools/profile_case.py channel128 6 > gpurun_out/prof/ncu_aa.log 2>&1; echo ncu_aa=$?
python tools/ncu_summary.py gpurun_out/prof/ncu_step_kernel.json channel3d_128=gpurun_out/prof/full_channel128.ncu-rep ras256_phi02=gpurun_out/prof/full_ras256_phi02.ncu-rep ras256_phi05=gpurun_out/prof/full_ras256_phi05.ncu-rep cavity2d_4096_a4=gpurun_out/prof/full_cavity2d_4096_a4.ncu-rep channel3d_128_f32=gpurun_out/prof/full_channel128_f32.ncu-rep channel3d_128_mrt=gpurun_out/prof/full_channel128_mrt.ncu-rep channel3d_128_aa_phase1=gpurun_out/prof/full_channel128_aa.ncu-rep@0 channel3d_128_aa_phase2=gpurun_out/prof/full_channel128_aa.ncu-rep@1 > gpurun_out/prof/ncu_summary.log 2>&1; echo summary=$?
for c in channel128 ras256_phi02 ras256_phi05 cavity2d_4096_a4; do
  ncu -i gpurun_out/prof/full_$c.ncu-rep --page raw --csv > gpurun_out/prof/raw_$c.csv 2>/dev/null
done
rm -f gpurun_out/prof/full_ras256_phi05.ncu-rep gpurun_out/prof/full_cavity2d_4096_a4.ncu-rep gpurun_out/prof/full_ras256_phi02.ncu-rep gpurun_out/prof/full_channel128_f32.ncu-rep gpurun_out/prof/full_channel128_mrt.ncu-rep gpurun_out/prof/full_channel128_aa.ncu-rep
du -sh gpurun_out
timeout 900 python bench.py --config ras1024 --phi 0.2 --steps 20 --warmup 4 > gpurun_out/prof/ras1024_phi02.json.log 2>&1; echo big02=$?
timeout 900 python bench.py --config ras1024 --phi 0.5 --single-copy --steps 20 --warmup 4 > gpurun_out/prof/ras1024_phi05_aa.json.log 2>&1; echo big05=$?
timeout 900 python bench.py --config ras1024 --phi 0.8 --single-copy --steps 20 --warmup 4 > gpurun_out/prof/ras1024_phi08_aa.json.log 2>&1; echo big08=$?
for a in "2 128" "4 128" "1 128 asym" "2 128 asym"; do timeout 300 python tools/slab_overhead.py $a 2>&1 | tail -1; done > gpurun_out/prof/slab_overhead.txt
tail -3 gpurun_out/prof/pytest_gpu.log

#!/bin/bash
# Round 2, first GPU session: parity suite (incl. 1000-step full-size goldens, multi-GPU ordering
# paths), default bench (with configs[4] point), FMA-variant A/B, 1024^3 lines + ncu capture,
# a 2-rank slab bench on one GPU (configs4_strong plumbing at 512^3).
mkdir -p gpurun_out/r2a
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2a/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r2a/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2a/bench.json.log 2>&1; echo bench=$?
tail -c 600 gpurun_out/r2a/bench.json.log
timeout 900 python tools/ab.py '{"rn": {}, "fma": {"LIB": "variants/lib_fma.so"}}' channel128 ras256_phi02 ras256_phi05 vessel4096 --rounds 5 --steps 64 > gpurun_out/r2a/ab_fma.log 2>&1; echo ab=$?
tail -12 gpurun_out/r2a/ab_fma.log
timeout 900 python tools/ab.py '{"rn": {"SPLBM_MODEL": "mrt"}, "fma": {"SPLBM_MODEL": "mrt", "LIB": "variants/lib_fma.so"}}' channel128 ras256_phi05 --rounds 5 --steps 64 > gpurun_out/r2a/ab_fma_mrt.log 2>&1; echo abmrt=$?
tail -6 gpurun_out/r2a/ab_fma_mrt.log
timeout 900 python bench.py --config ras1024 --phi 0.2 --steps 20 --warmup 4 > gpurun_out/r2a/ras1024_phi02.json.log 2>&1; echo big02=$?
SPLBM_LIB=variants/lib_fma.so timeout 900 python bench.py --config ras1024 --phi 0.2 --steps 20 --warmup 4 > gpurun_out/r2a/ras1024_phi02_fma.json.log 2>&1; echo big02fma=$?
timeout 900 python bench.py --config ras1024 --phi 0.2 --steps 20 --warmup 4 > gpurun_out/r2a/ras1024_phi02_b.json.log 2>&1; echo big02b=$?
timeout 1500 ncu --set full --replay-mode application --clock-control none --cache-control none --import-source on -k regex:t2c_step -s 4 -c 1 -o gpurun_out/r2a/full_ras1024_phi02 python tools/profile_case.py ras1024_phi02 6 > gpurun_out/r2a/ncu_ras1024.log 2>&1; echo ncu1024=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:t2c_step -s 4 -c 1 -o gpurun_out/r2a/full_ras256_phi02 python tools/profile_case.py ras256_phi02 6 > gpurun_out/r2a/ncu_ras256.log 2>&1; echo ncu256=$?
for c in ras1024_phi02 ras256_phi02; do ncu -i gpurun_out/r2a/full_$c.ncu-rep --page raw --csv > gpurun_out/r2a/raw_$c.csv 2>/dev/null; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 4 --c4-size 512 > gpurun_out/r2a/bench_n2_shared.json.log 2>&1; echo benchn2=$?
tail -c 1500 gpurun_out/r2a/bench_n2_shared.json.log
du -sh gpurun_out/r2a
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --cache-control all --csv --log-file gpurun_out/r2a/tma_probe.csv ./tools/tma_probe > gpurun_out/r2a/tma_probe.log 2>&1; echo tmaprobe=$?
./tools/tma_probe >> gpurun_out/r2a/tma_probe.log 2>&1

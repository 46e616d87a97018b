#!/bin/bash
# Round 2 (third session): configs[4] single-copy lines with the phase-1 register diet, the
# compute-sanitizer round (incl. the resident kernel), and bench.py --gpus 2 under torchrun with
# both ranks on this one GPU (validation of the N>1 path; configs[4] strong scaling at 256^3).
O=gpurun_out/r2o
mkdir -p $O
cd "$(dirname "$0")/.."
for phi in 0.5 0.8; do
  timeout 900 python bench.py --config ras1024 --phi $phi --single-copy --steps 200 --warmup 10 > $O/ras1024_phi${phi}_aa.json 2> $O/ras1024_phi${phi}_aa.err; echo big$phi=$?
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --c4-size 256 > $O/bench_n2.json 2> $O/bench_n2.err; echo n2=$?
tail -c 1500 $O/bench_n2.json
bash tools/sanitize_round.sh > $O/sanitizer.txt 2>&1; echo san=$?
cat $O/sanitizer.txt

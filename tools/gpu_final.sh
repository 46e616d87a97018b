#!/bin/bash
# Round 2 final check, as the driver runs it: smoke, GPU suite, bench N=1, reference arm, and
# bench --gpus 2 under torchrun (both ranks on this GPU; 256^3 configs[4] strong-scaling key).
O=gpurun_out/final
mkdir -p $O
cd "$(dirname "$0")/.."
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest=$?; tail -1 $O/pytest.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo benchref=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 20 --warmup 3 --c4-size 256 > $O/bench_n2.json 2> $O/bench_n2.err; echo n2=$?
tail -c 400 $O/bench_n2.json

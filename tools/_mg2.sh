mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --config ras1024 --phi 0.2 --gpus 2 --steps 10 --warmup 3 > gpurun_out/mg2.log 2>&1; echo rc=$?
grep metric gpurun_out/mg2.log | cut -c1-900; tail -3 gpurun_out/mg2.log | cut -c1-300
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/mg2b.log 2>&1; echo rc=$?
grep metric gpurun_out/mg2b.log | cut -c1-400

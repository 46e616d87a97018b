timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu6.log 2>&1; echo pytest=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/bench6_tr.log 2>&1; echo benchtr=$?

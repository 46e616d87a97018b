mkdir -p gpurun_out
for n in 1 2 3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 50 --warmup 5 > gpurun_out/mg1_$n.log 2>&1; echo n$n=$?
grep metric gpurun_out/mg1_$n.log | cut -c1-1500
done
SPLBM_SLAB_TRANSPORT=nccl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/mg1_nccl.log 2>&1; echo nccl=$?
tail -3 gpurun_out/mg1_nccl.log | cut -c1-600

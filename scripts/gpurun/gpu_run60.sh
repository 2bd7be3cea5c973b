cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# NCCL combine path per allreduce algorithm; per-collective
# syntax so torch's own broadcasts keep their default algorithm
port=29980
for algo in allreduce:tree allreduce:ring allreduce:nvls allreduce:nvlstree; do
port=$((port+1))
tag=${algo#allreduce:}
NCCL_ALGO=$algo NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=TUNING timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 50 --warmup 5 --combine nccl > gpurun_out/b60_4_nccl_$tag.log 2>&1
done
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# bench line with the new memory / one-thread CPU fields, N=1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/b59_1.log 2>&1
# NCCL combine path under each NCCL algorithm, N=4, cfg3
port=29970
for algo in auto Tree Ring NVLS; do
port=$((port+1))
if [ $algo = auto ]; then unset NCCL_ALGO; else export NCCL_ALGO=$algo; fi
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=TUNING timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 50 --warmup 5 --combine nccl > gpurun_out/b59_4_nccl_$algo.log 2>&1
done
unset NCCL_ALGO
port=$((port+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 50 --warmup 5 --combine p2p > gpurun_out/b59_4_p2p.log 2>&1
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/b1.log 2>&1
port=29760
for n in 2 4; do
for c in nccl p2p; do
port=$((port+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --steps 30 --warmup 5 --combine $c > gpurun_out/b${n}_$c.log 2>&1
done
done
port=$((port+1))
TD_POOL_FRAC=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 30 --warmup 5 --combine p2p > gpurun_out/b4_p2p_nopool.log 2>&1
port=$((port+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 30 --warmup 5 --combine p2p --seq-len 524288 > gpurun_out/b4_p2p_512k.log 2>&1
port=$((port+1))
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port scripts/sweep.py > gpurun_out/sweep4.log 2>&1
echo done

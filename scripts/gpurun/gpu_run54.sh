cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/final4_b1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --seq-len 131072 --no-cpu-baseline > gpurun_out/final4_b1_131k.log 2>&1
port=29700
for n in 2 4; do
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n > gpurun_out/final4_b$n.log 2>&1
done
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --seq-len 524288 --steps 100 > gpurun_out/final4_b4_512k.log 2>&1
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --combine nccl > gpurun_out/final4_b4_nccl.log 2>&1
echo done

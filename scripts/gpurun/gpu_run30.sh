cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload cfg4 --steps 20 > gpurun_out/w_cfg4_1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload cfg2 --steps 20 > gpurun_out/w_cfg2_1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload cfg1 --steps 20 > gpurun_out/w_cfg1_1.log 2>&1
port=29890
for n in 2 4; do
for algo in tree ring; do
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --workload cfg2 --algo $algo --steps 20 > gpurun_out/w_cfg2_${algo}_$n.log 2>&1
done
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --workload cfg4 --steps 20 > gpurun_out/w_cfg4_$n.log 2>&1
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --algo ring --steps 10 > gpurun_out/w_cfg3_ring_$n.log 2>&1
done
echo done

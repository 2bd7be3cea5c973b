cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r77
O=gpurun_out/r77
timeout 700 python -m pytest tests -q -m gpu -p timeout --timeout 500 > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
port=29800
for n in 2 4; do
port=$((port+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n > $O/b$n.log 2>&1
done
port=$((port+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 100 --seq-len 524288 > $O/b4_512k.log 2>&1
port=$((port+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --combine nccl > $O/b4_nccl.log 2>&1
port=$((port+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --workload cfg4 --steps 20 > $O/b4_cfg4.log 2>&1
timeout 300 python bench.py --workload cfg4 --steps 20 --warmup 3 --no-cpu-baseline > $O/b1_cfg4.log 2>&1
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -p timeout --timeout 800 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --phases --no-cpu-baseline > gpurun_out/b1.log 2>&1
timeout 300 python scripts/ts_probe.py > gpurun_out/ts1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29799 scripts/sweep.py --seq 65536,262144,1048576 > gpurun_out/sweep2.log 2>&1
port=29750
for n in 2 4; do
for c in nccl p2p; do
port=$((port+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --steps 20 --warmup 3 --phases --combine $c > gpurun_out/b${n}_$c.log 2>&1
done
done
port=$((port+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port scripts/ts_probe.py --combine p2p > gpurun_out/ts4_p2p.log 2>&1
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
port=29900
for v in 0; do
port=$((port+1))
TD_XCHG_VARIANT=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port scripts/xchg_probe.py > gpurun_out/xp_$v.log 2>&1
done
port=$((port+1))
PROBE_N=1048576 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port scripts/xchg_probe.py > gpurun_out/xp_big.log 2>&1
echo done
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p timeout --timeout 800 > gpurun_out/multi.log 2>&1
port=$((port+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 20 --warmup 3 --combine p2p > gpurun_out/b4_p2p.log 2>&1

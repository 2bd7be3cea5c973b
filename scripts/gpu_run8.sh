cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
port=29900
for v in 0 1 2 3 4; do
port=$((port+1))
TD_XCHG_VARIANT=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port scripts/xchg_probe.py > gpurun_out/xp_$v.log 2>&1
done
port=$((port+1))
PROBE_N=1048576 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port scripts/xchg_probe.py > gpurun_out/xp_big.log 2>&1
echo done

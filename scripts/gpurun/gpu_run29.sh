cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
port=29870
for rep in 1 2 3; do
for pull in 0 1; do
port=$((port+1))
TD_XCHG_PULL=$pull timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 100 --warmup 10 --seq-len 524288 > gpurun_out/ab_pull${pull}_$rep.log 2>&1
done; done

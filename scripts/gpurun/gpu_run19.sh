cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 4 --steps 30 --warmup 5 --combine p2p --seq-len 524288 > gpurun_out/b4_512k.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29814 scripts/ts_probe.py --seq-len 524288 --combine p2p > gpurun_out/ts4.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29816 bench.py --gpus 2 --steps 30 --warmup 5 --combine p2p --seq-len 262144 > gpurun_out/b2_256k.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "4 or 2" > gpurun_out/multi4.log 2>&1
echo "rc=$?" >> gpurun_out/multi4.log

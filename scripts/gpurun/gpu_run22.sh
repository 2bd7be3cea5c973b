cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TD_DEBUG_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29821 scripts/timeline_probe.py --seq-len 524288 > gpurun_out/tl4.log 2>&1
TD_XCHG_PULL=1 TD_DEBUG_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29822 scripts/timeline_probe.py --seq-len 524288 > gpurun_out/tl4_pull.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 4 --steps 30 --warmup 5 --combine p2p --seq-len 524288 > gpurun_out/b4_512k.log 2>&1
TD_XCHG_PULL=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29813 bench.py --gpus 4 --steps 30 --warmup 5 --combine p2p --seq-len 524288 > gpurun_out/b4_512k_pull.log 2>&1
TD_XCHG_PULL=1 timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "4" > gpurun_out/multi4.log 2>&1
echo "rc=$?" >> gpurun_out/multi4.log

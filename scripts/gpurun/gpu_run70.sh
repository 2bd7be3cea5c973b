cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TD_DEBUG_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29881 scripts/timeline_probe.py --seq-len 524288 --steps 30 > gpurun_out/tl70_4.log 2>&1
TD_DEBUG_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29882 scripts/timeline_probe.py --seq-len 262144 --steps 30 > gpurun_out/tl70_2.log 2>&1
TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 30 > gpurun_out/tl70_1.log 2>&1
echo done

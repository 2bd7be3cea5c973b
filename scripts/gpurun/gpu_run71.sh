cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TD_XCHG_PULL=1 TD_DEBUG_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29883 scripts/timeline_probe.py --seq-len 524288 --steps 30 > gpurun_out/tl71_4pull.log 2>&1
TD_DEBUG_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29884 scripts/timeline_probe.py --seq-len 524288 --steps 30 > gpurun_out/tl71_4push.log 2>&1
echo done

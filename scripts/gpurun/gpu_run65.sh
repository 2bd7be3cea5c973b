cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts65_1.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29878 scripts/ts_probe.py --seq-len 524288 > gpurun_out/ts65_4.log 2>&1
TD_DEBUG_TIMELINE=1 TL_DUMP_CTAS=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 20 > gpurun_out/tl65_1.log 2>&1
TD_DEBUG_TIMELINE=1 TL_DUMP_CTAS=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29879 scripts/timeline_probe.py --seq-len 524288 --steps 20 > gpurun_out/tl65_4.log 2>&1
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TD_DEBUG_TIMELINE=1 TL_DUMP_CTAS=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 20 > gpurun_out/tl64_1.log 2>&1
TD_DEBUG_TIMELINE=1 TL_DUMP_CTAS=1 TD_K1_PREFETCH=0 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 20 > gpurun_out/tl64_1_nopf.log 2>&1
TD_DEBUG_TIMELINE=1 TL_DUMP_CTAS=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29877 scripts/timeline_probe.py --seq-len 524288 --steps 20 > gpurun_out/tl64_4.log 2>&1
NOFLUSH=1 timeout 120 scripts/_bin/read_probe 536.9 > gpurun_out/rp64.log 2>&1
echo done

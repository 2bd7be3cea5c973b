cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TS_DUMP_CTAS=1 timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts_fwd.log 2>&1
TS_DUMP_CTAS=1 TD_DEBUG_REVERSE=1 timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts_rev.log 2>&1
TS_DUMP_CTAS=1 timeout 300 python scripts/ts_probe.py --seq-len 1048576 > gpurun_out/ts_fwd_1m.log 2>&1
echo done

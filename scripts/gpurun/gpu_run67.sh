cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts67.log 2>&1
timeout 300 python scripts/ts_probe.py --seq-len 16384 > gpurun_out/ts67_16k.log 2>&1
echo done

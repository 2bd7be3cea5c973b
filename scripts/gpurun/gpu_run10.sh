cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/ts_probe.py > gpurun_out/ts1.log 2>&1
timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts1_131k.log 2>&1
PROBE_N=1048576 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29971 scripts/xchg_probe.py > gpurun_out/xp_big.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --seq-len 131072 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_bf16|k2_combine" -s 10 -c 2 -o gpurun_out/prof_p8shard python bench.py --steps 2 --warmup 3 --no-cpu-baseline --seq-len 131072 > gpurun_out/ncu_full.log 2>&1
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/ts_probe.py --combine nccl > gpurun_out/ts1.log 2>&1
for c in p2p nccl; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2971$RANDOM bench.py --gpus 4 --steps 2 --warmup 1 --no-cpu-baseline --combine $c > /dev/null 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2972$((RANDOM%100)) scripts/ts_probe.py --combine $c > gpurun_out/ts4_$c.log 2>&1
done
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_bf16|k2_combine" -s 6 -c 2 -o gpurun_out/prof_k1k2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done

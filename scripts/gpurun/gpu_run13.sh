cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p timeout --timeout 800 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for f in 0 0.1 0.15 0.25; do
TD_POOL_FRAC=$f timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts_pool_$f.log 2>&1
TD_POOL_FRAC=$f timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --seq-len 131072 > gpurun_out/b131_pool_$f.log 2>&1
TD_POOL_FRAC=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b1m_pool_$f.log 2>&1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29981 bench.py --gpus 2 --steps 30 --warmup 5 --combine p2p > gpurun_out/b2_p2p.log 2>&1
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p timeout --timeout 800 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --phases --no-cpu-baseline > gpurun_out/b1.log 2>&1
for n in 2 4; do
for c in nccl p2p; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 296$n$((RANDOM%10)) bench.py --gpus $n --steps 20 --warmup 3 --phases --combine $c > gpurun_out/b${n}_$c.log 2>&1
done
done
echo done

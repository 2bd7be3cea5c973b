cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu4.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/final3_b1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final3_ref1.log 2>&1
port=29980
for n in 2 4; do
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n > gpurun_out/final3_b$n.log 2>&1
done
echo done

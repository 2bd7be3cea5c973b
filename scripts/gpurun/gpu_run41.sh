cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi.log 2>&1
echo "rc=$?" >> gpurun_out/multi.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29991 bench.py --gpus 4 --steps 50 --seq-len 524288 > gpurun_out/b4_512k.log 2>&1

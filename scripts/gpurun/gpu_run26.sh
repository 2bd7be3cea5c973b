cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu4.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/final_b1.log 2>&1
port=29850
for n in 2 4; do
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n > gpurun_out/final_b$n.log 2>&1
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref$n.log 2>&1
done
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --combine nccl > gpurun_out/final_b4_nccl.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/final_launches_131k.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --seq-len 131072 > gpurun_out/final_ncu_l.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_bf16|k2_combine" -s 10 -c 2 -o gpurun_out/final_prof_131k python bench.py --steps 2 --warmup 3 --no-cpu-baseline --seq-len 131072 > gpurun_out/final_ncu_f.log 2>&1
echo done

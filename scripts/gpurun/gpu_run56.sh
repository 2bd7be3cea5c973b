cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export TD_FUSED_TAIL=1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_fused.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_fused.log
export CUDA_VISIBLE_DEVICES=0
for v in "TD_FUSED_TAIL=1" "TD_FUSED_TAIL=0"; do
echo "$v" >> gpurun_out/ab_fused.log
env $v timeout 300 python bench.py --steps 50 --seq-len 131072 --no-cpu-baseline >> gpurun_out/ab_fused.log 2>&1
env $v TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 >> gpurun_out/ab_fused.log 2>&1
done
unset CUDA_VISIBLE_DEVICES
for v in "TD_FUSED_TAIL=1" "TD_FUSED_TAIL=0"; do
echo "$v" >> gpurun_out/ab_fused4.log
env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29721 bench.py --gpus 4 --steps 100 --seq-len 524288 >> gpurun_out/ab_fused4.log 2>&1
done

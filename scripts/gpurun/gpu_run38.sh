cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
export CUDA_VISIBLE_DEVICES=0
for v in "X=0" "TD_STEAL_SLOTS=0"; do
echo "$v" >> gpurun_out/ab_steal3.log
env $v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --seq-len 131072 >> gpurun_out/ab_steal3.log 2>&1
env $v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline >> gpurun_out/ab_steal3.log 2>&1
env $v timeout 300 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --workload cfg4 >> gpurun_out/ab_steal3.log 2>&1
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1
echo "rc=$?" >> gpurun_out/par.log
for i in 1 2 3 4; do
timeout 300 python bench.py --steps 30 --seq-len 131072 --no-cpu-baseline >> gpurun_out/cal131.log 2>&1
done
for i in 1 2; do
timeout 300 python bench.py --steps 20 --no-cpu-baseline >> gpurun_out/cal1m.log 2>&1
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
export CUDA_VISIBLE_DEVICES=0
timeout 600 python scripts/decode_loop.py --seq-len 1048576 > gpurun_out/loop1.log 2>&1
timeout 600 python scripts/decode_loop.py --seq-len 131072 >> gpurun_out/loop1.log 2>&1
timeout 300 python bench.py --steps 30 --seq-len 131072 --no-cpu-baseline > gpurun_out/b131.log 2>&1

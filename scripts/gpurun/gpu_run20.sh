cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/b1_default.log 2>&1
echo "rc=$?" >> gpurun_out/b1_default.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/b1_ref.log 2>&1
echo "rc=$?" >> gpurun_out/b1_ref.log

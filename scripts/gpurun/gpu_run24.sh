cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_energy.py -x -q > gpurun_out/energy.log 2>&1
echo "rc=$?" >> gpurun_out/energy.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "2" > gpurun_out/multi2.log 2>&1
echo "rc=$?" >> gpurun_out/multi2.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1
echo "rc=$?" >> gpurun_out/par.log

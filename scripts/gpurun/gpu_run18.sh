cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 300 scripts/_bin/read_probe > gpurun_out/read_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "4" > gpurun_out/multi4.log 2>&1
echo "rc=$?" >> gpurun_out/multi4.log

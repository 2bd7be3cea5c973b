cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
STEPS=30 timeout 300 python -X faulthandler scripts/append_repro2.py > gpurun_out/app1.log 2>&1
echo "rc=$?" >> gpurun_out/app1.log
timeout 600 python -X faulthandler -m pytest tests/test_gpu_parity.py -x -q -k "append or place_matches" > gpurun_out/app3.log 2>&1
echo "rc=$?" >> gpurun_out/app3.log

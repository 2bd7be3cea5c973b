cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_capi_c.py -q -s > gpurun_out/capi_c.log 2>&1
echo "rc=$?" >> gpurun_out/capi_c.log

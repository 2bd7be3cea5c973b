cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1
echo "rc=$?" >> gpurun_out/par.log
TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 1048576 --steps 40 --append > gpurun_out/tl_app2.log 2>&1
TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 40 --append >> gpurun_out/tl_app2.log 2>&1
timeout 600 python scripts/decode_loop.py --seq-len 1048576 > gpurun_out/loop1.log 2>&1
timeout 600 python scripts/decode_loop.py --seq-len 131072 >> gpurun_out/loop1.log 2>&1

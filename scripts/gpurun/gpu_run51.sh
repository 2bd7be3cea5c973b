cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 128 --append > gpurun_out/tl_app6.log 2>&1
timeout 600 python scripts/decode_loop.py --seq-len 131072 --steps 128 > gpurun_out/loop1.log 2>&1
timeout 600 python scripts/decode_loop.py --seq-len 131072 --steps 28 >> gpurun_out/loop1.log 2>&1

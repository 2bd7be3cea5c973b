cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
timeout 600 python scripts/decode_loop.py --seq-len 1048576 > gpurun_out/loop1.log 2>&1
TD_STEAL_SLOTS=0 timeout 600 python scripts/decode_loop.py --seq-len 1048576 >> gpurun_out/loop1.log 2>&1
TD_CALIBRATE=0 timeout 600 python scripts/decode_loop.py --seq-len 1048576 >> gpurun_out/loop1.log 2>&1
timeout 600 python scripts/decode_loop.py --seq-len 131072 >> gpurun_out/loop1.log 2>&1

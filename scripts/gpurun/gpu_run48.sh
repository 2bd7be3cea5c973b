cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
timeout 600 python scripts/decode_loop.py --seq-len 131072 --steps 128 > gpurun_out/loop1.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
for i in 1 2 3; do
TL_DUMP_CTAS=1 TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 10 >> gpurun_out/tl_ctas131.log 2>&1
done

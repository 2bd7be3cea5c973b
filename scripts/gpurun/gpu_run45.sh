cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
for v in "X=0" "TD_STEAL_SLOTS=0" "TD_CALIBRATE=0"; do
echo "$v" >> gpurun_out/tl_app.log
env $v TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 1048576 --steps 40 --append >> gpurun_out/tl_app.log 2>&1
env $v TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 1048576 --steps 40 >> gpurun_out/tl_app.log 2>&1
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
for v in "X=0" "TD_SM_AFFINITY=0" "TD_CALIBRATE=0" "TD_K1_PDL=0"; do
echo "$v" >> gpurun_out/tl_app4.log
env $v TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 60 --append >> gpurun_out/tl_app4.log 2>&1
env $v TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 60 >> gpurun_out/tl_app4.log 2>&1
done

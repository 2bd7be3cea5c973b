cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
for rep in 1 2; do
for v in "TD_STEAL_SLOTS=0" "TD_STEAL_SLOTS=4" "TD_STEAL_SLOTS=8" "TD_STEAL_SLOTS=12"; do
echo "$v" >> gpurun_out/ab_steal2.log
env $v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --seq-len 131072 >> gpurun_out/ab_steal2.log 2>&1
env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/ab_steal2.log 2>&1
done; done
TD_STEAL_SLOTS=8 TL_DUMP_CTAS=1 TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 10 > gpurun_out/tl_steal.log 2>&1
TD_STEAL_SLOTS=0 TL_DUMP_CTAS=1 TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 10 >> gpurun_out/tl_steal.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
for rep in 1 2; do
for v in "X=0" "TD_K2_WARPS=1" "TD_K2_WARPS=1 TD_K2_MAX_BLOCKS=4096" "TD_K1_PDL=0" "TD_K1_EARLY_TRIGGER=1"; do
echo "$v" >> gpurun_out/ab_k2.log
env $v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --seq-len 131072 >> gpurun_out/ab_k2.log 2>&1
env $v timeout 300 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --workload cfg4 >> gpurun_out/ab_k2.log 2>&1
done; done

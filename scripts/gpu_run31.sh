cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --b 16 --nq 64 --nkv 8 --seq-len 131072 > gpurun_out/tl_cfg4.log 2>&1
TD_DEBUG_TIMELINE=1 TD_K1_PDL=0 timeout 300 python scripts/timeline_probe.py --b 16 --nq 64 --nkv 8 --seq-len 131072 >> gpurun_out/tl_cfg4.log 2>&1
TD_K1_PDL=0 timeout 600 python bench.py --workload cfg4 --steps 20 --no-cpu-baseline > gpurun_out/w_cfg4_nopdl.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py > gpurun_out/tl.log 2>&1
TD_DEBUG_TIMELINE=1 TD_K1_PDL=0 timeout 300 python scripts/timeline_probe.py >> gpurun_out/tl.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --seq-len 131072 > gpurun_out/b1_131k.log 2>&1
TD_K1_PDL=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --seq-len 131072 > gpurun_out/b1_131k_nopdl.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b1_1m.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par.log 2>&1
echo "rc=$?" >> gpurun_out/par.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_energy.py -x -q > gpurun_out/par.log 2>&1
echo "rc=$?" >> gpurun_out/par.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --seq-len 131072 > gpurun_out/b1_131k.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --workload cfg1 > gpurun_out/b1_cfg1.log 2>&1

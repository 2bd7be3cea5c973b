cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
timeout 300 python bench.py --workload cfg1 --seq-len 4194304 --steps 20 --no-cpu-baseline > gpurun_out/f32_4m.log 2>&1
timeout 300 python bench.py --workload cfg1 --seq-len 1048576 --steps 20 --no-cpu-baseline > gpurun_out/f32_1m.log 2>&1
timeout 300 python bench.py --workload cfg1 --steps 30 --no-cpu-baseline > gpurun_out/f32_64k.log 2>&1

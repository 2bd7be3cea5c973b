cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
export CUDA_VISIBLE_DEVICES=0
timeout 300 python bench.py > gpurun_out/b1_default.log 2>&1
echo "bench rc=$?" >> gpurun_out/b1_default.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --seq-len 131072 > gpurun_out/b1_131k.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_1m.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_131k.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --seq-len 131072 > gpurun_out/ncu_l2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_bf16|k2_combine" -s 10 -c 2 -o gpurun_out/prof_1m python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_f1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_bf16|k2_combine" -s 10 -c 2 -o gpurun_out/prof_131k python bench.py --steps 2 --warmup 3 --no-cpu-baseline --seq-len 131072 > gpurun_out/ncu_f2.log 2>&1
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "append" -p timeout --timeout 500 > gpurun_out/pytest62.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest62.log
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/b62_1m.log 2>&1 && \
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r62_launches_1m.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r62_ncu_l1m.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_bf16|k2_combine" -s 30 -c 2 -o gpurun_out/r62_prof_1m python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r62_ncu_f1m.log 2>&1
echo done

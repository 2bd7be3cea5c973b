cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r76
O=gpurun_out/r76
timeout 600 python -m pytest tests -q -m gpu -p timeout --timeout 400 > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 400 python bench.py > $O/b1.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 5 --seq-len 131072 --no-cpu-baseline > $O/b1_131k.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_1m.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_l1m.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k1_bf16|k2_combine" -s 30 -c 2 -o $O/prof_131k python bench.py --steps 2 --warmup 3 --seq-len 131072 --no-cpu-baseline > $O/ncu_f131k.log 2>&1
echo done

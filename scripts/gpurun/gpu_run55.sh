cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29831 scripts/sweep.py --out gpurun_out/sweepf_p4.csv > gpurun_out/sweepf4.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29832 scripts/sweep.py --out gpurun_out/sweepf_p2.csv > gpurun_out/sweepf2.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python scripts/sweep.py --out gpurun_out/sweepf_p1.csv > gpurun_out/sweepf1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/final_launches_1m.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_l1m.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_bf16|k2_combine" -s 30 -c 2 -o gpurun_out/final_prof_1m python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_f1m.log 2>&1
echo done

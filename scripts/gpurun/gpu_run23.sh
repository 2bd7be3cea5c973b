cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29831 scripts/sweep.py --out gpurun_out/sweep_p4.csv > gpurun_out/sweep4.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29832 scripts/sweep.py --out gpurun_out/sweep_p2.csv > gpurun_out/sweep2.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python scripts/sweep.py --out gpurun_out/sweep_p1.csv > gpurun_out/sweep1.log 2>&1
echo done

# 16K-4M sweep (configs[4]) at 1/2/4 GPUs (one 4-GPU box)
set -x
O=gpurun_out/sw2; mkdir -p $O
T="timeout 1200 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 1200 python scripts/sweep.py --out $O/r2_sweep_p1.csv > $O/r2_sweep_p1.jsonl 2>>$O/err.log
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29703 scripts/sweep.py --out $O/r2_sweep_p2.csv > $O/r2_sweep_p2.jsonl 2>>$O/err.log
CUDA_VISIBLE_DEVICES=0,1,2,3 $T --nproc-per-node 4 --master-port 29704 scripts/sweep.py --out $O/r2_sweep_p4.csv > $O/r2_sweep_p4.jsonl 2>>$O/err.log
ls -la $O

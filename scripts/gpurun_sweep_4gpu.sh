# 16K-4M sweep (configs[4]) at 1/2/4 GPUs (one 4-GPU box), plus the cfg1 line (flushed L2)
set -x
O=gpurun_out/sw3; mkdir -p $O
T="timeout 1200 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --workload cfg1 --steps 30 > $O/b1_cfg1.json 2>>$O/err.log
CUDA_VISIBLE_DEVICES=0 timeout 1200 python scripts/sweep.py --out $O/r2_sweep_p1.csv > $O/r2_sweep_p1.jsonl 2>>$O/err.log
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29703 scripts/sweep.py --out $O/r2_sweep_p2.csv > $O/r2_sweep_p2.jsonl 2>>$O/err.log
CUDA_VISIBLE_DEVICES=0,1,2,3 $T --nproc-per-node 4 --master-port 29704 scripts/sweep.py --out $O/r2_sweep_p4.csv > $O/r2_sweep_p4.jsonl 2>>$O/err.log
CUDA_VISIBLE_DEVICES=0,1,2,3 $T --nproc-per-node 4 --master-port 29705 bench.py --gpus 4 --seq-len 65536 --steps 30 > $O/b4_64k.json 2>>$O/err.log
ls -la $O

# The round-2 final multi-GPU set (one 4-GPU box): N=2 on GPUs 0,1, then N=4.
set -x
O=gpurun_out/fin4; mkdir -p $O
T="timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
export CUDA_VISIBLE_DEVICES=0,1
$T --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > $O/b2.json 2>>$O/err.log
$T --nproc-per-node 2 --master-port 29602 bench.py --gpus 2 --workload cfg2 --steps 20 > $O/b2_cfg2.json 2>>$O/err.log
$T --nproc-per-node 2 --master-port 29603 bench.py --gpus 2 --impl reference --steps 3 --warmup 1 > $O/ref2.json 2>>$O/err.log
$T --nproc-per-node 2 --master-port 29604 scripts/decode_loop.py --seq-len 262144 > $O/dl2_256k.json 2>>$O/err.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k2_exchange --launch-skip 1 --launch-count 1 --metrics nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum -o $O/ncu_k2x_2gpu python scripts/k2x_profile.py > $O/ncu_k2x.log 2>&1
export CUDA_VISIBLE_DEVICES=0,1,2,3
$T --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 > $O/b4.json 2>>$O/err.log
$T --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --seq-len 524288 > $O/b4_512k.json 2>>$O/err.log
$T --nproc-per-node 4 --master-port 29613 bench.py --gpus 4 --workload cfg2 --steps 20 > $O/b4_cfg2.json 2>>$O/err.log
$T --nproc-per-node 4 --master-port 29614 bench.py --gpus 4 --workload cfg4 --steps 20 > $O/b4_cfg4.json 2>>$O/err.log
$T --nproc-per-node 4 --master-port 29615 bench.py --gpus 4 --combine nccl_device --no-compare > $O/b4_nccl_device.json 2>>$O/err.log
$T --nproc-per-node 4 --master-port 29616 bench.py --gpus 4 --impl reference --steps 3 --warmup 1 > $O/ref4.json 2>>$O/err.log
(timeout 900 python -m pytest tests -m gpu -q > $O/pytest_4gpu.log 2>&1; echo pytest rc=$? >> $O/pytest_4gpu.log)
ls -la $O

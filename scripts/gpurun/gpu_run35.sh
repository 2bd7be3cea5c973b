cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TD_DEBUG_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29961 scripts/timeline_probe.py --seq-len 524288 > gpurun_out/tlv_base.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29962 bench.py --gpus 4 --steps 100 --seq-len 524288 > gpurun_out/bv_base.log 2>&1
cp paper_2408_04093_b200/_variants/libtreedec_b200_gpuld.so paper_2408_04093_b200/libtreedec_b200.so
TD_DEBUG_TIMELINE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29963 scripts/timeline_probe.py --seq-len 524288 > gpurun_out/tlv_gpuld.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29964 bench.py --gpus 4 --steps 100 --seq-len 524288 > gpurun_out/bv_gpuld.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "4" > gpurun_out/multi_gpuld.log 2>&1
echo "rc=$?" >> gpurun_out/multi_gpuld.log

O=gpurun_out/sp2; mkdir -p $O
for r in 1 2 3; do for p in 0 2; do CUDA_VISIBLE_DEVICES=0 TD_K2_STREAM_POLL=$p timeout 150 python bench.py --seq-len 131072 --steps 50 > $O/b131k_p${p}_r$r.json 2>>$O/err.log; done; done
for p in 0 2; do CUDA_VISIBLE_DEVICES=0 TD_K2_STREAM_POLL=$p TD_DEBUG_TIMELINE=1 timeout 150 python scripts/timeline_probe.py --steps 40 > $O/tl_p$p.log 2>&1; done
T="timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
for r in 1 2; do for p in 0 2; do TD_K2_STREAM_POLL=$p $T --master-port 2970$r bench.py --gpus 4 --seq-len 524288 --steps 50 --no-compare > $O/b4_512k_p${p}_r$r.json 2>>$O/err.log; done; done
CUDA_VISIBLE_DEVICES=0 TD_K2_STREAM_POLL=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "stream or determin or worker" > $O/pytest_p2.log 2>&1
TD_K2_STREAM_POLL=2 timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_multi_p2.log 2>&1

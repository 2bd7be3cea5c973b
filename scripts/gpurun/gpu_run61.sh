cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# K1 prefetch before the PDL wait: A/B (TD_K1_PREFETCH=0 is the previous kernel)
for rep in 1 2; do
for pf in 0 1; do
TD_K1_PREFETCH=$pf timeout 300 python bench.py --steps 100 --warmup 5 --seq-len 131072 --no-cpu-baseline > gpurun_out/b61_131k_pf${pf}_$rep.log 2>&1
TD_K1_PREFETCH=$pf timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b61_1m_pf${pf}_$rep.log 2>&1
done
done
port=29990
for rep in 1 2; do
for pf in 0 1; do
port=$((port+1))
TD_K1_PREFETCH=$pf timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 100 --warmup 5 --seq-len 524288 > gpurun_out/b61_4x131k_pf${pf}_$rep.log 2>&1
done
done
timeout 300 python scripts/decode_loop.py --seq-len 131072 --steps 64 > gpurun_out/b61_loop.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p timeout --timeout 800 > gpurun_out/pytest_gpu61.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu61.log
echo done

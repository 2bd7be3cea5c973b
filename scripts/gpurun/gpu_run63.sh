cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# extra L2 prefetch before the PDL wait: A/B over TD_K1_L2_PREFETCH
for rep in 1 2; do
for l2 in 0 3 6 12; do
TD_K1_L2_PREFETCH=$l2 timeout 300 python bench.py --steps 100 --warmup 5 --seq-len 131072 --no-cpu-baseline > gpurun_out/b63_131k_l2${l2}_${rep}.log 2>&1
grep '^{' gpurun_out/b63_131k_l2${l2}_${rep}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('131k', $l2, $rep, d['value'])" >> gpurun_out/b63_summary.txt
done
done
port=29990
for rep in 1 2; do
for l2 in 0 3 6 12; do
port=$((port+1))
TD_K1_L2_PREFETCH=$l2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 100 --warmup 5 --seq-len 524288 --no-cpu-baseline > gpurun_out/b63_4x_l2${l2}_$rep.log 2>&1
grep '^{' gpurun_out/b63_4x_l2${l2}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('4x131k', $l2, $rep, d['value'])" >> gpurun_out/b63_summary.txt
done
done
for l2 in 0 6; do
TD_K1_L2_PREFETCH=$l2 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b63_1m_l2$l2.log 2>&1
grep '^{' gpurun_out/b63_1m_l2$l2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('1m', $l2, 1, d['value'])" >> gpurun_out/b63_summary.txt
done
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# A/B of K1's batched epilogue merge (TD_DEBUG_REVERSE=2: the previous cta_merge)
for r in 0 2; do
TD_DEBUG_REVERSE=$r timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts69_r$r.log 2>&1
TD_DEBUG_REVERSE=$r TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 20 > gpurun_out/tl69_r$r.log 2>&1
done
for rep in 1 2 3; do
for r in 0 2; do
TD_DEBUG_REVERSE=$r timeout 300 python bench.py --steps 100 --warmup 5 --seq-len 131072 --no-cpu-baseline > gpurun_out/b69_131k_r${r}_$rep.log 2>&1
grep '^{' gpurun_out/b69_131k_r${r}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('131k', $r, $rep, d['value'])" >> gpurun_out/b69_summary.txt
done
done
port=29990
for rep in 1 2; do
for r in 0 2; do
port=$((port+1))
TD_DEBUG_REVERSE=$r timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 100 --warmup 5 --seq-len 524288 --no-cpu-baseline > gpurun_out/b69_4x_r${r}_$rep.log 2>&1
grep '^{' gpurun_out/b69_4x_r${r}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('4x131k', $r, $rep, d['value'])" >> gpurun_out/b69_summary.txt
done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p timeout --timeout 500 > gpurun_out/pytest69.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest69.log
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -p timeout --timeout 600 > gpurun_out/pytest73.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest73.log
for k in 0 1; do
TD_K1_COUNT=$k TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 20 > gpurun_out/tl73_k$k.log 2>&1
done
for rep in 1 2 3; do
for k in 0 1; do
TD_K1_COUNT=$k timeout 300 python bench.py --steps 100 --warmup 5 --seq-len 131072 --no-cpu-baseline > gpurun_out/b73_131k_k${k}_$rep.log 2>&1
grep '^{' gpurun_out/b73_131k_k${k}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('131k', $k, $rep, d['value'], d['e2e']['matches_device_output'])" >> gpurun_out/b73_summary.txt
done
done
port=29990
for rep in 1 2; do
for k in 0 1; do
port=$((port+1))
TD_K1_COUNT=$k timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 100 --warmup 5 --seq-len 524288 --no-cpu-baseline > gpurun_out/b73_4x_k${k}_$rep.log 2>&1
grep '^{' gpurun_out/b73_4x_k${k}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('4x131k', $k, $rep, d['value'], d['e2e']['matches_device_output'])" >> gpurun_out/b73_summary.txt
done
done
for k in 0 1; do
TD_K1_COUNT=$k timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/b73_1m_k$k.log 2>&1
grep '^{' gpurun_out/b73_1m_k$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('1m', $k, 1, d['value'], d['e2e']['matches_device_output'])" >> gpurun_out/b73_summary.txt
done
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -p timeout --timeout 700 > gpurun_out/pytest75.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest75.log
port=29990
for rep in 1 2 3; do
for c in 0 4; do
port=$((port+1))
TD_K2_COLS=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 100 --warmup 5 --seq-len 524288 --no-cpu-baseline > gpurun_out/b75_4x_c${c}_$rep.log 2>&1
grep '^{' gpurun_out/b75_4x_c${c}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('4x131k', $c, $rep, d['value'], d['e2e']['matches_device_output'])" >> gpurun_out/b75_summary.txt
done
done
for c in 0 4; do
port=$((port+1))
TD_K2_COLS=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 2 --steps 100 --warmup 5 --seq-len 262144 --no-cpu-baseline > gpurun_out/b75_2x_c${c}.log 2>&1
grep '^{' gpurun_out/b75_2x_c${c}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('2x131k', $c, 1, d['value'], d['e2e']['matches_device_output'])" >> gpurun_out/b75_summary.txt
done
echo done

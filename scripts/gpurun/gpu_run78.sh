cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r78
O=gpurun_out/r78
port=29900
for rep in 1 2; do
for c in 0 4; do
port=$((port+1))
TD_K2_COLS=$c timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --workload cfg4 --steps 20 --no-cpu-baseline > $O/cfg4_c${c}_$rep.log 2>&1
grep '^{' $O/cfg4_c${c}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 n4 cols', $c, 'rep', $rep, d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])" >> $O/summary.txt
done
done
echo done

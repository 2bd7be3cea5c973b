cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in 0 1; do
TD_K2_WARM=$w timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts66_w$w.log 2>&1
TD_K2_WARM=$w TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 20 > gpurun_out/tl66_w$w.log 2>&1
done
for rep in 1 2; do
for w in 0 1; do
TD_K2_WARM=$w timeout 300 python bench.py --steps 100 --warmup 5 --seq-len 131072 --no-cpu-baseline > gpurun_out/b66_131k_w${w}_$rep.log 2>&1
grep '^{' gpurun_out/b66_131k_w${w}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('131k', $w, $rep, d['value'])" >> gpurun_out/b66_summary.txt
done
done
port=29990
for rep in 1 2; do
for w in 0 1; do
port=$((port+1))
TD_K2_WARM=$w timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 100 --warmup 5 --seq-len 524288 --no-cpu-baseline > gpurun_out/b66_4x_w${w}_$rep.log 2>&1
grep '^{' gpurun_out/b66_4x_w${w}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('4x131k', $w, $rep, d['value'])" >> gpurun_out/b66_summary.txt
done
done
echo done

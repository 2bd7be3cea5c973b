cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for f in 0 1; do
TD_K2_FAST=$f timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts68_f$f.log 2>&1
TD_K2_FAST=$f TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 20 > gpurun_out/tl68_f$f.log 2>&1
done
for rep in 1 2; do
for f in 0 1; do
TD_K2_FAST=$f timeout 300 python bench.py --steps 100 --warmup 5 --seq-len 131072 --no-cpu-baseline > gpurun_out/b68_131k_f${f}_$rep.log 2>&1
grep '^{' gpurun_out/b68_131k_f${f}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('131k', $f, $rep, d['value'])" >> gpurun_out/b68_summary.txt
done
done
port=29990
for rep in 1 2; do
for f in 0 1; do
port=$((port+1))
TD_K2_FAST=$f timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 100 --warmup 5 --seq-len 524288 --no-cpu-baseline > gpurun_out/b68_4x_f${f}_$rep.log 2>&1
grep '^{' gpurun_out/b68_4x_f${f}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('4x131k', $f, $rep, d['value'])" >> gpurun_out/b68_summary.txt
done
done
timeout 900 python -m pytest tests -q -m gpu -x -p timeout --timeout 600 > gpurun_out/pytest68.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest68.log
echo done

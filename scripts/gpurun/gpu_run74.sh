cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capi_c.py tests/test_gpu_shim.py -q -m gpu -x -p timeout --timeout 600 > gpurun_out/pytest74.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest74.log
for c in 0 4; do
TD_K2_COLS=$c TD_DEBUG_TIMELINE=1 timeout 300 python scripts/timeline_probe.py --seq-len 131072 --steps 20 > gpurun_out/tl74_c$c.log 2>&1
done
for rep in 1 2 3; do
for c in 0 4; do
TD_K2_COLS=$c timeout 300 python bench.py --steps 100 --warmup 5 --seq-len 131072 --no-cpu-baseline > gpurun_out/b74_131k_c${c}_$rep.log 2>&1
grep '^{' gpurun_out/b74_131k_c${c}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('131k', $c, $rep, d['value'], d['e2e']['matches_device_output'])" >> gpurun_out/b74_summary.txt
done
done
echo done

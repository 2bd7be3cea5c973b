cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p timeout --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for f in 0 0.1 0.15 0.25; do
TD_POOL_FRAC=$f timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts_pool_$f.log 2>&1
TD_POOL_FRAC=$f timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --seq-len 131072 > gpurun_out/b131_pool_$f.log 2>&1
TD_POOL_FRAC=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b1m_pool_$f.log 2>&1
done
echo done

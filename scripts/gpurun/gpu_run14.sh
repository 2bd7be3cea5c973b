cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p timeout --timeout 800 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in "TD_CALIBRATE=0 TD_POOL_FRAC=0" "TD_CALIBRATE=1 TD_POOL_FRAC=0" "TD_CALIBRATE=1 TD_POOL_FRAC=0.05" "TD_CALIBRATE=1 TD_POOL_FRAC=0.15"; do
tag=$(echo $cfg | tr ' =' '_-')
env $cfg timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts_$tag.log 2>&1
env $cfg timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --seq-len 131072 > gpurun_out/b131_$tag.log 2>&1
env $cfg timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b1m_$tag.log 2>&1
done
echo done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
TS_DUMP_CTAS=1 timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts_ctas.log 2>&1
TS_DUMP_CTAS=1 TD_POOL_FRAC=0.3 timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts_ctas_p30.log 2>&1
TS_DUMP_CTAS=1 TD_POOL_CHUNK=1 timeout 300 python scripts/ts_probe.py --seq-len 131072 > gpurun_out/ts_ctas_c1.log 2>&1
for f in 0.05 0.15 0.3; do for c in 1 2 4; do
TD_POOL_FRAC=$f TD_POOL_CHUNK=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --seq-len 131072 > gpurun_out/b131_f${f}_c$c.log 2>&1
done; done
